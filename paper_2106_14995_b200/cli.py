"""Command-line front end (SPEC.md `cli` module).

    python -m paper_2106_14995_b200 --mode bench --n 8 --batch 10000 --out runs/
    python -m paper_2106_14995_b200 --mode admm --case case9.m --max-iter 5000 --out runs/

bench: solves `batch` copies of hs45(n) on the device; writes bench.csv
(problem, status, iterations, f_star, time_s) and bench.json (total time,
throughput, failures); exit 0 iff every problem converged.
admm:  parses a MATPOWER case, runs the device ADMM until both residuals meet
their tolerances or max-iter; writes admm.csv (iter, primal, dual, objective,
step_time_s, stage_time_s and, with --workers G >= 2, batch_time_p0..p{G-1}:
each contiguous partition's share of that iteration's branch stage solved
alone) and admm.json (status, iterations, objective, residuals,
ImbalanceStats over all iterations' partition times); exit 0 iff converged, 1
otherwise.  Usage and parse errors exit 2.  Timing columns are the
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
    G = a.workers
    parts = np.array_split(np.arange(case.grid.n_branch), G) if G >= 2 else None
    lo, up = A.branch_bounds(case.grid, opts.branch_dim)
    part_times = []  # [iteration][partition] seconds
    tsolver = None
    if parts is not None:
        from . import Solver

        tsolver = Solver((0,))
    with open(os.path.join(a.out, "admm.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["iter", "primal", "dual", "objective", "step_time_s", "stage_time_s"] +
                   ([f"batch_time_p{q}" for q in range(G)] if parts is not None else []))
        for k in range(1, a.max_iter + 1):
            if parts is not None:  # the stage's inputs: warm starts and multipliers before the step
                x0, prm = solver.get(A.BRANCH_X), solver.get(A.BRANCH_PARAMS)
            t0 = time.perf_counter()
            p, d = solver.step()
            dt = time.perf_counter() - t0
            stage = solver.stage_times()[0]
            obj = case.cost(solver.get(A.GEN_P))
            row = [k, repr(p), repr(d), repr(obj), f"{dt:.9f}", f"{stage:.9f}"]
            if parts is not None:
                pt = A.partition_stage_times(tsolver, x0, prm, lo, up, parts)
                part_times.append(pt)
                row += [f"{v:.9f}" for v in pt]
            w.writerow(row)
            if p <= a.tol_primal and d <= a.tol_dual:
                break
    converged = p <= a.tol_primal and d <= a.tol_dual
    summary = {"mode": "admm", "case": os.path.basename(a.case), "status": "converged" if converged else "max_iter",
               "iterations": k, "objective": case.cost(solver.get(A.GEN_P)), "primal": p, "dual": d,
               "n_bus": case.grid.n_bus, "n_gen": case.grid.n_gen, "n_branch": case.grid.n_branch,
               "line_limits": bool(a.line_limits)}
    if a.line_limits:
        summary["max_line_violation"] = float(solver.get(A.LINE_VIOL)[0])
    # ImbalanceStats (batch.hpp:80-111) over every
    # iteration's per-partition batch times: each contiguous partition's share
    # of that iteration's branch stage solved alone from the same inputs
    if part_times:
        im = imbalance(part_times)
        summary["imbalance"] = {"nu_max": im.nu_max, "nu_min": im.nu_min, "nu_mean": im.nu_mean,
                                "partitions": G, "iterations": len(part_times),
                                "partition": "contiguous even (batch.hpp:61-70)"}
        tsolver.close()
    solver.close()
    with open(os.path.join(a.out, "admm.json"), "w") as f:
        json.dump(summary, f, indent=1)
    return EXIT_OK if converged else EXIT_NOT_CONVERGED


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
