"""Command-line front end (SPEC.md `cli` module).

    python -m paper_2106_14995_b200 --mode bench --n 8 --batch 10000 --out runs/
    python -m paper_2106_14995_b200 --mode admm --case case9.m --max-iter 5000 --out runs/

bench: solves `batch` copies of hs45(n) on the device; writes bench.csv
(problem, status, iterations, f_star, time_s) and bench.json (total time,
throughput, failures); exit 0 iff every problem converged.
admm:  parses a MATPOWER case, runs the device ADMM until both residuals meet
their tolerances or max-iter; writes admm.csv (iter, primal, dual, objective,
step_time_s) and admm.json (status, iterations, objective, residuals,
imbalance over the `workers` partitions of the last branch stage); exit 0 iff
converged, 1 otherwise.  Usage and parse errors exit 2.  Timing columns are the
only non-deterministic outputs.
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import sys
import time

EXIT_OK, EXIT_NOT_CONVERGED, EXIT_USAGE = 0, 1, 2


class UsageError(Exception):
    pass


def _parser():
    ap = argparse.ArgumentParser(prog="python -m paper_2106_14995_b200", description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--mode", choices=["bench", "admm"], required=True)
    ap.add_argument("--case", help="MATPOWER case file (admm)")
    ap.add_argument("--n", type=int, default=8, help="hs45 dimension (bench), 1..64")
    ap.add_argument("--batch", type=int, default=10000, help="number of hs45 problems (bench)")
    ap.add_argument("--workers", type=int, default=1, help="GPUs (bench partitions) / imbalance partitions (admm)")
    ap.add_argument("--rho0", type=float, default=10.0, help="ADMM rho for power couplings (4 rho0 for voltage)")
    ap.add_argument("--max-iter", type=int, default=5000)
    ap.add_argument("--tol-primal", type=float, default=1e-4)
    ap.add_argument("--tol-dual", type=float, default=1e-3)
    ap.add_argument("--tol-pg", type=float, default=1e-6, help="TronConfig.tol_pg")
    ap.add_argument("--line-limits", action="store_true", help="enforce rateA (d=6 branch subproblems)")
    ap.add_argument("--out", default=".", help="output directory")
    ap.add_argument("--seed", type=int, default=0, help="reserved (the hs45 batch is deterministic)")
    return ap


class _ArgParser(argparse.ArgumentParser):
    def error(self, message):
        raise UsageError(message)


def run_bench(a) -> int:
    import numpy as np

    from . import Solver, TronConfig, imbalance, synth

    if not (1 <= a.n <= 64):
        raise UsageError(f"--n {a.n}: hs45 dimension out of capacity [1, 64] (batch.hpp kDefaultCapacity)")
    if a.batch < 0 or a.workers < 1:
        raise UsageError("--batch must be >= 0 and --workers >= 1")
    b = synth.hs45(a.batch, a.n)
    solver = Solver(tuple(range(a.workers)))
    t0 = time.perf_counter()
    r = solver.solve_batch(b, cfg=TronConfig(tol_pg=a.tol_pg))
    wall = time.perf_counter() - t0
    solver.close()
    st = np.asarray(r.status)
    os.makedirs(a.out, exist_ok=True)
    with open(os.path.join(a.out, "bench.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["problem", "status", "iterations", "f_star", "time_s"])
        for k in range(a.batch):
            w.writerow([k, int(st[k]), int(r.iterations[k]), repr(float(r.f_star[k])),
                        f"{float(r.per_problem_time[k]):.9f}"])
    fails = int(np.sum(st != 0))
    summary = {"mode": "bench", "n": a.n, "batch": a.batch, "workers": a.workers, "total_time_s": wall,
               "throughput_solves_per_s": (a.batch / wall) if wall > 0 else None, "failures": fails,
               "partition_times_s": list(r.partition_times)}
    if a.workers >= 2 and a.batch > 0:
        im = imbalance([list(r.partition_times)])
        summary["imbalance"] = {"nu_max": im.nu_max, "nu_min": im.nu_min, "nu_mean": im.nu_mean}
    with open(os.path.join(a.out, "bench.json"), "w") as f:
        json.dump(summary, f, indent=1)
    return EXIT_OK if fails == 0 else EXIT_NOT_CONVERGED


def run_admm(a) -> int:
    import numpy as np

    from . import TronConfig, imbalance
    from . import admm as A
    from . import matpower

    if not a.case:
        raise UsageError("--mode admm needs --case")
    if not os.path.isfile(a.case):
        raise UsageError(f"--case {a.case}: no such file")
    if a.max_iter < 1 or not (a.rho0 > 0) or a.workers < 1:
        raise UsageError("--max-iter, --rho0 and --workers must be positive")
    try:
        case = matpower.load(a.case)
    except matpower.MatpowerError as e:
        raise UsageError(f"{a.case}: {e}") from None
    opts = A.AdmmOptions(rho_pq=a.rho0, rho_va=4.0 * a.rho0, tron=TronConfig(tol_pg=a.tol_pg),
                         line_limits=a.line_limits)
    solver = A.AdmmSolver(case.grid, opts)
    os.makedirs(a.out, exist_ok=True)
    p = d = float("inf")
    k = 0
    with open(os.path.join(a.out, "admm.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["iter", "primal", "dual", "objective", "step_time_s"])
        for k in range(1, a.max_iter + 1):
            t0 = time.perf_counter()
            p, d = solver.step()
            dt = time.perf_counter() - t0
            obj = case.cost(solver.get(A.GEN_P))
            w.writerow([k, repr(p), repr(d), repr(obj), f"{dt:.9f}"])
            if p <= a.tol_primal and d <= a.tol_dual:
                break
    converged = p <= a.tol_primal and d <= a.tol_dual
    summary = {"mode": "admm", "case": os.path.basename(a.case), "status": "converged" if converged else "max_iter",
               "iterations": k, "objective": case.cost(solver.get(A.GEN_P)), "primal": p, "dual": d,
               "n_bus": case.grid.n_bus, "n_gen": case.grid.n_gen, "n_branch": case.grid.n_branch,
               "line_limits": bool(a.line_limits)}
    if a.line_limits:
        summary["max_line_violation"] = float(solver.get(A.LINE_VIOL)[0])
    # imbalance (PAPER §5.3) of the last branch stage over `workers` contiguous
    # partitions, partition time = summed per-branch device time
    if a.workers >= 2:
        t = _branch_times(solver, case, opts)
        parts = np.array_split(t, a.workers)
        im = imbalance([[float(np.sum(q)) for q in parts]])
        summary["imbalance"] = {"nu_max": im.nu_max, "nu_min": im.nu_min, "nu_mean": im.nu_mean,
                                "partitions": a.workers}
    solver.close()
    with open(os.path.join(a.out, "admm.json"), "w") as f:
        json.dump(summary, f, indent=1)
    return EXIT_OK if converged else EXIT_NOT_CONVERGED


def _branch_times(solver, case, opts):
    """Per-branch device times of one more branch solve at the current state."""
    import numpy as np

    from . import ProblemBatch, Solver
    from . import admm as A

    g = case.grid
    D = opts.branch_dim
    x = solver.get(A.BRANCH_X)
    prm = solver.get(A.BRANCH_PARAMS)
    lo = np.stack([g.bus_vmin[g.br_from], g.bus_vmin[g.br_to], np.full(g.n_branch, -2 * np.pi),
                   np.full(g.n_branch, -2 * np.pi)], 1)
    up = np.stack([g.bus_vmax[g.br_from], g.bus_vmax[g.br_to], np.full(g.n_branch, 2 * np.pi),
                   np.full(g.n_branch, 2 * np.pi)], 1)
    if D == 6:
        sm = np.where(np.isfinite(prm[:, 35]), prm[:, 35], np.inf)
        lo = np.concatenate([lo, -np.stack([sm, sm], 1)], 1)
        up = np.concatenate([up, np.zeros((g.n_branch, 2))], 1)
    s = Solver((0,))
    r = s.solve_batch(ProblemBatch(3, D, lo, up, prm, x))
    s.close()
    return np.asarray(r.per_problem_time)


def main(argv=None) -> int:
    ap = _parser()
    ap.__class__ = _ArgParser
    try:
        a = ap.parse_args(argv)
        return run_bench(a) if a.mode == "bench" else run_admm(a)
    except UsageError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
