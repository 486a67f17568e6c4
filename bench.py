#!/usr/bin/env python
"""Benchmark of the batched TRON hot path (BASELINE.json configs[1], C2):
65,536 synthetic AC-OPF branch augmented-Lagrangian subproblems (d = 6) per GPU.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one batched solve of the whole per-GPU batch (weak scaling: every
rank solves its own 65,536-problem batch; no collective on the data path).
Prints ONE JSON line on rank 0.

value : solves/s over all ranks, inputs resident in HBM, device time of the
        solve kernel (CUDA events on the launching stream, L2 flushed between
        steps outside the timed events), max over ranks.
e2e   : same metric through the public API with pinned HOST buffers
        (H2D of x0/l/u/params + kernel + D2H of every SolveReport field).
--impl reference : the reference's own CPU solve_batch (the unmodified
        reference headers compiled into oracle/_ref/libtronref.so, all host
        threads) on a bounded sample of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

BATCH = 65536
DIM = 6
METRIC = "bound-constrained solves/sec (batch, FP64)"
WORKLOAD = "C2: 65,536 synthetic AC-OPF branch augmented-Lagrangian subproblems (d=6) per GPU"



def kernel_form(d, count):
    """Which device kernel the library routes a (dim, count) ncvx batch to
    under KernelForm.AUTO (csrc/tron_kernels.cuh resolve_form)."""
    if d == 4 and count >= 8192:
        return "thread per problem"
    if d <= 16:
        return "warp per problem"
    return f"block of {32 if d <= 32 else 64 if d <= 64 else 128} threads (persistent)"

def sig(x, digits=5):
    """Round floats in a nested structure to `digits` significant digits
    (keeps the ADMM block short enough for the driver's 1,500-char tail)."""
    if isinstance(x, float):
        return float(f"{x:.{digits}g}")
    if isinstance(x, dict):
        return {k: sig(v, digits) for k, v in x.items()}
    if isinstance(x, (list, tuple)):
        return [sig(v, digits) for v in x]
    return x


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """SM clocks and throttle reasons sampled (NVML, every 20 ms) DURING the
    timed region; falls back to nvidia-smi if NVML is unavailable."""

    # NVML clocks-event-reason bits
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, device: int):
        self.device = device
        self.rows = []  # (sm_mhz, max_mhz, reasons_bitmask)
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((sm, mx, rs))
                self._stop.wait(0.02)
            return
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                                      "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                sm, mx, rs = [c.strip() for c in out.split(",")]
                self.rows.append((float(sm), float(mx), int(rs, 16)))
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.05)  # first sample before the timed region starts
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({name for _, _, rs in self.rows for bit, name in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows)}


def cpu_reference_run(batch, workers, reps=1):
    """The reference's own solve_batch (oracle/_ref) on `batch`; returns
    (solves/s best of reps, wall seconds)."""
    from oracle import pyoracle

    best = 0.0
    total = 0.0
    for _ in range(reps):
        t0 = time.perf_counter()
        r = pyoracle.solve_batch(batch, impl="ref", workers=workers)
        dt = time.perf_counter() - t0
        total += dt
        assert r.rc == 0, f"reference solve_batch threw: {pyoracle.last_error()}"
        best = max(best, batch.count / r.batch_wall_time)
    return best, total


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_sample(full_batch, seconds_target=1.5, workers=1, rate_guess=15000.0):
    from paper_2106_14995_b200 import ProblemBatch

    n = int(min(full_batch.count, max(256, seconds_target * rate_guess * workers)))
    return ProblemBatch(full_batch.family, full_batch.dim, full_batch.lower[:n], full_batch.upper[:n],
                        full_batch.params[:n], full_batch.x0[:n]), n


def c2_config(n, world):
    """The C2 workload description shared by both arms' JSON lines."""
    return {"workload": WORKLOAD, "family": "branch", "dim": DIM, "batch_per_gpu": n, "global_batch": world * n,
            "seed": "2+rank", "parallelism": f"batch sharded over {world} GPU(s)",
            "l2": "flushed (256 MiB write) between timed steps, outside the events", "mode": "exact"}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return 0
    from oracle import pyoracle
    from paper_2106_14995_b200 import synth

    if not pyoracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtronref.so not built (needs /root/reference at build time)"}))
        return 0
    cores = os.cpu_count() or 1
    full = synth.branch(BATCH, DIM, seed=2)
    sample, n = cpu_sample(full, seconds_target=2.0, workers=cores)
    for _ in range(max(1, args.warmup)):
        cpu_reference_run(sample, cores)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, _ = cpu_reference_run(sample, cores)
        vals.append(v)
    wall = time.perf_counter() - t0
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(c2_config(BATCH, world), l2="n/a (host CPU)",
                       parallelism=f"reference solve_batch, std::thread over {cores} host cores"),
        "cpu_baseline": {"value": value, "unit": "solves/s", "cores": cores, "kind": "reference",
                         "sample": f"first {n} of the {BATCH} C2 problems per step, reference solve_batch(workers={cores})"},
        "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def c5_grid():
    from paper_2106_14995_b200 import synth

    nb = int(round(70000 * 13659 / 20467))  # C4's bus / branch ratio: 46,716 buses
    return synth.grid(nb, 70000, int(0.3 * nb))


def replay_imbalance(grid, dev, iters=5, parts=(2, 4, 8)):
    """SPEC.md:408 / PAPER.md:689-703 per-GPU imbalance of the C5 branch stage
    at G = 2 / 4 / 8, measured on one GPU: before each of `iters` ADMM
    iterations the branch stage's inputs (warm starts, multipliers) are
    snapshotted and every partition's share is solved alone
    (admm.partition_stage_times: its kernel time = what one GPU of a G-GPU run
    spends on the stage).  Contiguous even partitions (batch.hpp:61-70, the
    paper's dispatch) against a cost-aware one (LPT over the per-branch TRON
    iteration counts of the PREVIOUS iteration's stage, PAPER.md:715 future
    work)."""
    import torch

    from paper_2106_14995_b200 import ProblemBatch, Solver, imbalance
    from paper_2106_14995_b200 import admm as A

    run = A.AdmmSolver(grid, device=dev.index)
    for _ in range(3):
        run.step()
    solver = Solver((dev.index,))
    n = grid.n_branch
    lo, up = A.branch_bounds(grid, 4)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    prev_cost = None
    times = {("contiguous", G): [] for G in parts}
    times.update({("cost_aware", G): [] for G in parts})
    for _ in range(iters):
        x, prm = run.get(A.BRANCH_X), run.get(A.BRANCH_PARAMS)
        full = Solver.alloc_result(n, 4, device=True)
        solver.solve_batch(ProblemBatch(3, 4, t(lo), t(up), t(prm), t(x)), out=full)
        # cost proxy: TRON iterations per branch (the thread form's per-problem
        # device time is its whole warp's lifetime, so it does not separate
        # the branches of one warp)
        cost = full.iterations.cpu().numpy().astype(np.float64)
        for G in parts:
            cut = [n * k // G for k in range(G + 1)]
            times[("contiguous", G)].append(A.partition_stage_times(
                solver, x, prm, lo, up, [np.arange(cut[k], cut[k + 1]) for k in range(G)], dev.index))
            if prev_cost is not None:  # LPT on last iteration's per-branch times
                order = np.argsort(-prev_cost, kind="stable")
                load = np.zeros(G)
                owner = np.empty(n, np.int64)
                for j in order:
                    k = int(np.argmin(load))
                    owner[j] = k
                    load[k] += prev_cost[j]
                times[("cost_aware", G)].append(A.partition_stage_times(
                    solver, x, prm, lo, up, [np.nonzero(owner == k)[0] for k in range(G)], dev.index))
        prev_cost = cost
        run.step()
    run.close()
    solver.close()
    out = {}
    for (kind, G), tt in times.items():
        if tt:
            st = imbalance(tt)
            out.setdefault(kind, {})[f"G{G}"] = {"nu_max": round(st.nu_max, 1), "nu_min": round(st.nu_min, 1),
                                                 "nu_mean": round(st.nu_mean, 1),
                                                 "max_part_ms": round(1e3 * max(max(r) for r in tt), 3)}
    out["method"] = ("one GPU, each partition's share of the C5 branch stage solved alone (kernel time) on "
                     f"{iters} successive ADMM iterations; cost-aware = LPT over the previous iteration's "
                     "per-branch TRON iteration counts")
    return out


def admm_summary(line):
    """The ADMM numbers without their descriptions (those are in admm_detail)."""
    if not line:
        return line
    out = {"metric": line["metric"], "value": line["value"], "unit": line["unit"],
           "ms_per_iter": line["ms_per_iter"], "workload": line["config"]["workload"]}
    for k in ("per_step", "line_limits", "cpu_baseline"):
        if isinstance(line.get(k), dict):
            out[k] = line[k].get("value")
    if "imbalance" in line:
        out["imbalance"] = {k: line["imbalance"][k] for k in ("nu_max", "nu_min", "nu_mean")}
    if "c5" in line:
        c5 = line["c5"]
        out["c5"] = {"value": c5["value"], "ms_per_iter": c5["ms_per_iter"]}
        rep = c5.get("imbalance_replay") or {}
        out["c5"]["nu_mean_contiguous_vs_cost_aware"] = {
            G: [rep.get("contiguous", {}).get(G, {}).get("nu_mean"), rep.get("cost_aware", {}).get(G, {}).get("nu_mean")]
            for G in ("G2", "G4", "G8")}
    return sig(out, 4)


def run_admm(args, rank, world, local, dev):
    """ADMM iterations/s.  N = 1: C4 (13,659 buses / 20,467 branches / 4,092
    gens) through tb_admm_run (one CUDA graph per iteration, device stop flag,
    no host round trip per iteration) and through the per-iteration blocking
    step, C4 with line limits, and C5 (70,000 branches, 46,716 buses) through
    the sharded driver at world 1 plus its replayed G = 2/4/8 imbalance.
    N > 1: C5 sharded over N GPUs (NCCL all-gather of the branch solutions +
    max-allreduce of the residuals per iteration), per-rank branch-stage times
    -> imbalance."""
    import torch
    import torch.distributed as dist

    from paper_2106_14995_b200 import admm as A
    from paper_2106_14995_b200 import imbalance, synth

    K = args.admm_iters
    W0 = max(3, args.warmup)

    def sharded_rate(grid, record):
        run = A.ShardedAdmm(grid, rank, world, local, record_times=record)
        for _ in range(W0):
            run.step()
        run._ev.clear()
        stream = torch.cuda.current_stream(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(K):
            run.step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return run, float(ms.item()) / K

    c5 = c5_grid()
    if world > 1:
        if not dist.is_initialized():
            return None
        run, ms_iter = sharded_rate(c5, True)
        pt = run.partition_times()
        st = imbalance(pt)
        return {"metric": "ADMM iterations/sec", "value": 1e3 / ms_iter, "unit": "iter/s", "ms_per_iter": ms_iter,
                "scaling": "strong", "iters_timed": K, "warmup_iters": W0,
                "config": {"workload": "C5", "n_bus": c5.n_bus, "n_branch": c5.n_branch, "n_gen": c5.n_gen,
                           "branch_dim": 4, "parallelism": f"branches sharded over {world} GPUs, NCCL all-gather"},
                "imbalance": {"nu_max": st.nu_max, "nu_min": st.nu_min, "nu_mean": st.nu_mean,
                              "partition": "contiguous even (batch.hpp:61-70)",
                              "stage_ms_per_rank_mean": [1e3 * float(np.mean(c)) for c in zip(*pt)]},
                "residuals_first_last": [run.history[0], run.history[-1]]}

    # ---- C4 on one GPU
    grid = synth.grid(13659, 20467, 4092)
    g_run = A.AdmmSolver(grid, device=local)
    g_run.run(W0)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    g_run.run(K)  # max_iter K, no tolerance: exactly K graph-replayed iterations
    dt_run = (time.perf_counter() - t0) / K
    g_run.close()
    step_run, ms_step = sharded_rate(grid, False)
    line = {"metric": "ADMM iterations/sec", "value": 1.0 / dt_run, "unit": "iter/s", "ms_per_iter": 1e3 * dt_run,
            "scaling": None, "iters_timed": K, "warmup_iters": W0,
            "timing": "host wall clock around tb_admm_run(K) (graph replay, one final sync)",
            "config": {"workload": "C4", "n_bus": grid.n_bus, "n_branch": grid.n_branch, "n_gen": grid.n_gen,
                       "branch_dim": 4, "parallelism": "1 GPU"},
            "per_step": {"value": 1e3 / ms_step, "ms_per_iter": ms_step,
                         "timing": "device events around K blocking sharded-driver steps (residual read-back each)"},
            "residuals_first_last": [step_run.history[0], step_run.history[-1]]}
    ll = A.AdmmSolver(grid, A.AdmmOptions(line_limits=True), local)
    ll.run(W0)
    r0 = int(ll.get(A.AUGLAG_ROUNDS)[0])
    k = max(5, K // 2)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    ll.run(k)
    dt = (time.perf_counter() - t0) / k
    line["line_limits"] = {
        "value": 1.0 / dt, "unit": "iter/s", "ms_per_iter": 1e3 * dt, "iters_timed": k,
        "auglag_rounds_per_iter": (int(ll.get(A.AUGLAG_ROUNDS)[0]) - r0) / k,
        "max_line_violation": float(ll.get(A.LINE_VIOL)[0]), "branch_dim": 6,
        "timing": "host wall clock around tb_admm_run(k) (branch stage = one fused augmented-Lagrangian launch)"}
    ll.close()
    if rank == 0 and not args.no_cpu_baseline:
        try:
            from oracle import pyoracle

            cores = os.cpu_count() or 1
            cpu = pyoracle.OracleAdmm(grid, workers=cores)
            cpu.step()
            t0 = time.perf_counter()
            for _ in range(3):
                cpu.step()
            v = 3 / (time.perf_counter() - t0)
            line["cpu_baseline"] = {"value": v, "unit": "iter/s", "cores": cores, "kind": "port",
                                    "sample": "iterations 2-4 of the same C4 ADMM run, oracle/admm_oracle.c "
                                              f"(branch stage through the C TRON restatement, {cores} threads)"}
        except Exception as e:
            line["cpu_baseline"] = {"value": None, "sample": f"failed: {e}"}
    # ---- C5 at N = 1 (the first point of the scaling curve) + replayed imbalance
    c5_run, ms5 = sharded_rate(c5, False)
    line["c5"] = {"value": 1e3 / ms5, "unit": "iter/s", "ms_per_iter": ms5, "iters_timed": K,
                  "config": {"workload": "C5", "n_bus": c5.n_bus, "n_branch": c5.n_branch, "n_gen": c5.n_gen,
                             "parallelism": "1 GPU, sharded driver at world 1"},
                  "residuals_first_last": [c5_run.history[0], c5_run.history[-1]]}
    del c5_run
    if not args.no_imbalance:
        try:
            line["c5"]["imbalance_replay"] = replay_imbalance(c5, dev)
        except Exception as e:
            line["c5"]["imbalance_replay"] = {"error": repr(e)}
    return line


C3_DIMS = (4, 8, 16, 32, 64, 128)
C3_BATCH = 32768


def run_sweep(args, dev, fp64_peak=None):
    """C1 (1,024 ncvx d=4) and the C3 dimension sweep (ncvx, batch 32,768,
    d = 4..128): device time of one batched solve with inputs in HBM (median
    of `reps` after a warm-up) next to the reference's CPU solve_batch on a
    bounded sample (all host threads).  Parity for these shapes is covered by
    tests/test_gpu_parity.py (bitwise); this reports speed only."""
    import torch

    from paper_2106_14995_b200 import ProblemBatch, Solver, synth

    solver = Solver((dev.index,))
    exec_solver = Solver((dev.index,), fast_forward=2)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    cores = os.cpu_count() or 1
    have_ref = False
    try:
        from oracle import pyoracle

        have_ref = pyoracle.ref_available() and not args.no_cpu_baseline
    except Exception:
        pass
    out = []
    cases = [("C1", 1024, 4, 1)] + [("C3", C3_BATCH, d, 3 + d) for d in C3_DIMS]
    for name, B, d, seed in cases:
        b = synth.ncvx(B, d, seed=seed)
        db = ProblemBatch(b.family, d, t(b.lower), t(b.upper), t(b.params), t(b.x0))
        out_d = Solver.alloc_result(B, d, device=True)
        solver.solve_batch(db, out=out_d)
        reps = 3 if d <= 64 else 2
        ks = []
        for _ in range(reps):
            solver.solve_batch(db, out=out_d)
            ks.append(out_d.kernel_time)
        ms = 1e3 * statistics.median(ks)
        # algorithmic flops EXECUTED on the same batch (untimed counting variant,
        # identical results; fast_forward=2 leaves out the skipped replays and
        # memoised factorizations)
        exec_solver.solve_batch(db, out=out_d, count_flops=True)
        flops = float(out_d.flops.sum().item())
        row = {"config": name, "family": "ncvx", "dim": d, "batch": B, "ms": ms, "solves_per_s": B / (ms * 1e-3),
               "achieved_tflops": flops / (ms * 1e-3) / 1e12, "flops_per_solve": flops / B,
               "kernel": kernel_form(d, B),
               "mean_iterations": float(out_d.iterations.double().mean().item()),
               "status_counts": {str(k): int(v) for k, v in
                                 zip(*np.unique(out_d.status.cpu().numpy(), return_counts=True))}}
        if have_ref:
            guess = {4: 60000, 8: 20000, 16: 6000, 32: 2500, 64: 700, 128: 200}[d]  # per-thread solves/s
            n = int(min(B, max(64, 1.0 * guess * cores)))
            sub = ProblemBatch(b.family, d, b.lower[:n], b.upper[:n], b.params[:n], b.x0[:n])
            v, _ = cpu_reference_run(sub, cores, reps=2)
            row["cpu_baseline"] = {"value": v, "unit": "solves/s", "cores": cores, "kind": "reference",
                                   "sample": f"first {n} of the {B} problems, reference solve_batch(workers={cores})"}
            row["speedup_vs_cpu"] = row["solves_per_s"] / v
        if fp64_peak:
            row["roofline_frac"] = row["achieved_tflops"] / fp64_peak
        out.append(row)
        del db, out_d, b
        torch.cuda.empty_cache()
    solver.close()
    exec_solver.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-admm", action="store_true")
    ap.add_argument("--admm-iters", type=int, default=20)
    ap.add_argument("--no-sweep", action="store_true", help="skip the C1 / C3 dimension sweep")
    ap.add_argument("--no-imbalance", action="store_true", help="skip the replayed C5 partition imbalance")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup) if args.impl == "ours" else args.warmup

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_2106_14995_b200 import Solver, TronConfig, _lib, synth

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    lib = _lib.load()
    solver = Solver((local,))
    cfg = TronConfig()
    batch = synth.branch(args.batch, DIM, seed=2 + rank)
    N = batch.count

    # ---- device-resident inputs (HBM) and outputs
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    from paper_2106_14995_b200 import ProblemBatch

    dbatch = ProblemBatch(batch.family, batch.dim, t(batch.lower), t(batch.upper), t(batch.params), t(batch.x0))
    dout = Solver.alloc_result(N, DIM, device=True)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    # a dedicated (non-default) stream: the kernel and the timing events are
    # enqueued on the same stream handle
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)

    def device_step():
        solver.solve_batch(dbatch, cfg=cfg, out=dout, stream=stream.cuda_stream)

    for _ in range(args.warmup):
        device_step()
    torch.cuda.synchronize(dev)

    # parity spot check (bitwise vs the CPU oracle) on the first 512 problems
    parity = None
    if rank == 0:
        try:
            from oracle import pyoracle

            m = min(512, N)
            sub = ProblemBatch(batch.family, DIM, batch.lower[:m], batch.upper[:m], batch.params[:m], batch.x0[:m])
            ref = pyoracle.solve_batch(sub, impl="oracle", workers=os.cpu_count() or 1)
            ok = all(np.array_equal(getattr(dout, k)[:m].cpu().numpy(), getattr(ref, k))
                     for k in ("x_star", "f_star", "pg_norm", "status", "iterations", "cg_iterations", "f_evals"))
            parity = f"bitwise {'match' if ok else 'MISMATCH'} vs CPU oracle on first {m} problems"
        except Exception as e:  # oracle not built on this box
            parity = f"not checked ({e})"

    # ---- timed region: device-resident
    launches0 = lib.tb_kernel_launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clocks:
        for k in range(args.steps):
            flush.random_(0, 255)  # untimed L2 flush between steps
            ev[k][0].record(stream)
            device_step()
            ev[k][1].record(stream)
        torch.cuda.synchronize(dev)
    barrier()
    launches = lib.tb_kernel_launch_count() - launches0
    ms_steps = [a.elapsed_time(b) for a, b in ev]
    ms_total = sum(ms_steps)
    mx = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    ms_total = float(mx.item())
    ms_per_step = ms_total / args.steps
    value = world * N / (ms_per_step * 1e-3)

    # ---- algorithmic flops per launch: one untimed run of the counting
    # variant (identical results; the count is deterministic)
    solver.solve_batch(dbatch, cfg=cfg, out=dout, stream=stream.cuda_stream, count_flops=True)
    torch.cuda.synchronize(dev)
    flops_per_launch = float(dout.flops.sum().item())  # the reference's count (skipped replays credited)
    status = dout.status.cpu().numpy()
    # executed flops: the fast-forwarded replays of a zero-change iteration are
    # not executed, so they do not count toward the achieved rate
    exec_solver = Solver((local,), fast_forward=2)
    exec_solver.solve_batch(dbatch, cfg=cfg, out=dout, stream=stream.cuda_stream, count_flops=True)
    torch.cuda.synchronize(dev)
    exec_flops = float(dout.flops.sum().item())
    exec_solver.close()
    achieved_tflops = exec_flops / (ms_per_step * 1e-3) / 1e12
    # the same timed steps with fast-forward off (every replay executed)
    nff = Solver((local,), fast_forward=False)
    for _ in range(2):
        nff.solve_batch(dbatch, cfg=cfg, out=dout, stream=stream.cuda_stream)
    evn = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize(dev)
    for k in range(args.steps):
        flush.random_(0, 255)
        evn[k][0].record(stream)
        nff.solve_batch(dbatch, cfg=cfg, out=dout, stream=stream.cuda_stream)
        evn[k][1].record(stream)
    torch.cuda.synchronize(dev)
    nff.close()
    ms_nff = statistics.median(a.elapsed_time(b) for a, b in evn)
    no_ff = {"value": world * N / (ms_nff * 1e-3), "ms_per_step": ms_nff,
             "note": "device time with fast_forward off (median step; every zero-change replay executed)"}
    peak = _lib.C.c_double()
    lib.tb_measure_fp64_peak(local, _lib.C.byref(peak))
    fp64_peak = peak.value

    # ---- e2e through the public API with pinned host buffers
    def pinned(a):
        p = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        p.copy_(torch.from_numpy(np.ascontiguousarray(a)))
        return p.numpy()

    hbatch = ProblemBatch(batch.family, DIM, pinned(batch.lower), pinned(batch.upper), pinned(batch.params),
                          pinned(batch.x0))
    hout = Solver.alloc_result(N, DIM, device=False)
    tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64}
    for name in ("x_star", "f_star", "pg_norm", "status", "iterations", "cg_iterations", "f_evals",
                 "per_problem_time", "flops"):
        a = getattr(hout, name)
        setattr(hout, name, torch.empty(a.shape, dtype=tdt[a.dtype], pin_memory=True).numpy())
    for _ in range(2):
        solver.solve_batch(hbatch, cfg=cfg, out=hout)
    barrier()
    e2e_times = []
    for _ in range(max(3, args.steps // 2)):
        t0 = time.perf_counter()
        solver.solve_batch(hbatch, cfg=cfg, out=hout)
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = statistics.median(e2e_times)
    e2e_t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = world * N / float(e2e_t.item())
    h2d = sum(a.nbytes for a in (hbatch.x0, hbatch.lower, hbatch.upper, hbatch.params))
    # every SolveReport field + per-problem device time (flops are not requested, so not copied)
    d2h = (hout.x_star.nbytes + hout.f_star.nbytes + hout.pg_norm.nbytes + hout.status.nbytes +
           hout.iterations.nbytes + hout.cg_iterations.nbytes + hout.f_evals.nbytes + hout.per_problem_time.nbytes)

    # ---- e2e with PAGEABLE host buffers (plain numpy: the library's pinned
    # staging + chunked pipeline) and through the C++ drop-in
    # (tronbatch::gpu::solve_batch, std::vector<BranchProblem> in, BatchResult out)
    pout = Solver.alloc_result(N, DIM, device=False)
    solver.solve_batch(batch, cfg=cfg, out=pout)
    pt = []
    for _ in range(max(3, args.steps // 4)):
        t0 = time.perf_counter()
        solver.solve_batch(batch, cfg=cfg, out=pout)
        pt.append(time.perf_counter() - t0)
    e2e_pageable = {"value": world * N / statistics.median(pt), "unit": "solves/s",
                    "note": "same call with pageable numpy buffers (library-owned pinned staging)"}
    dropin = None
    exe = os.path.join(ROOT, "oracle", "_ref", "gpu_dropin_bench")
    if rank == 0 and world == 1 and os.path.exists(exe):
        try:
            path = os.path.join("/tmp", f"tb_c2_batch_{os.getpid()}.bin")
            with open(path, "wb") as fh:
                fh.write(np.array([N, DIM, batch.params.shape[1]], dtype=np.int64).tobytes())
                for arr in (batch.x0, batch.lower, batch.upper, batch.params):
                    fh.write(np.ascontiguousarray(arr, dtype=np.float64).tobytes())
            out = subprocess.run([exe, path, "5"], capture_output=True, text=True, timeout=300)
            os.remove(path)
            dropin = json.loads(out.stdout.strip().splitlines()[-1])
            dropin["note"] = ("C++ drop-in tronbatch::gpu::solve_batch end to end: vector<BranchProblem> packing, "
                              "pinned staging, pipeline, 65,536 SolveReports (tests/cpp/gpu_dropin_bench.cpp); "
                              "value_incl_freeing_previous_result also times destroying the caller's previous "
                              "BatchResult (65,536 heap vectors) in `br = solve_batch(...)`")
        except Exception as e:
            dropin = {"value": None, "error": repr(e)}

    # ---- CPU baseline (rank 0, N=1 only): the reference's solve_batch
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import pyoracle

            if pyoracle.ref_available():
                cores = os.cpu_count() or 1
                sample, n = cpu_sample(batch, seconds_target=2.0, workers=cores)
                cpu_reference_run(sample, cores)
                v, _ = cpu_reference_run(sample, cores, reps=3)
                one, n1 = cpu_sample(batch, seconds_target=1.0, workers=1)
                v1, _ = cpu_reference_run(one, 1, reps=2)
                cpu = {"value": v, "unit": "solves/s", "cores": cores, "kind": "reference",
                       "sample": f"first {n} of the {N} C2 problems, reference solve_batch(workers={cores}), best of 3",
                       "cpu_model": cpu_model(), "single_thread_value": v1,
                       "single_thread_sample": f"first {n1} problems, workers=1, best of 2"}
        except Exception as e:
            cpu = {"value": None, "unit": "solves/s", "cores": None, "kind": "reference", "sample": f"failed: {e}"}

    admm_line = None
    if not args.no_admm:
        admm_line = run_admm(args, rank, world, local, dev)
    sweep = None
    if rank == 0 and world == 1 and not args.no_sweep:
        try:
            sweep = run_sweep(args, dev, fp64_peak)
        except Exception as e:
            sweep = [{"error": repr(e)}]

    traffic = None
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("bytes_per_launch")
        except Exception:
            traffic = None

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": c2_config(N, world),
            "e2e": {"value": e2e_value, "unit": "solves/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "e2e_pageable": e2e_pageable,
            "e2e_cpp_dropin": dropin,
            "roofline": {"bound": "fp64", "achieved": achieved_tflops, "peak": fp64_peak, "unit": "TFLOP/s",
                         "frac": achieved_tflops / fp64_peak if fp64_peak else None, "traffic": traffic,
                         "peak_source": "DFMA microbenchmark measured in this run (tb_measure_fp64_peak)",
                         "flops_per_launch": exec_flops,
                         "flops_per_launch_reference_count": flops_per_launch,
                         "flop_model": "algorithmic flops per SURVEY 8(d)/DESIGN.md, counted per problem on device; "
                                       "achieved uses the EXECUTED flops (fast-forwarded replays excluded); the "
                                       "reference count credits them"},
            "no_fast_forward": no_ff,
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
            "gpu_launches": int(launches),
            "launch_order": "ranked on the device by start projected-gradient norm (DESIGN.md 4g), inside the "
                            "timed region: 3 order kernels + 1 solve launch per step",
            "parity": parity,
            "status_counts": {str(k): int(v) for k, v in zip(*np.unique(status, return_counts=True))},
            "admm_detail": sig(admm_line),
            "sweep": sweep,
            "ms_per_step_all": ms_steps,
            "admm": admm_summary(admm_line),  # last and short: the driver keeps the line's 1,500-char tail
        }
        print(json.dumps(line), flush=True)
    solver.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
