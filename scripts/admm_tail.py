"""Per-branch latency distribution of the ADMM branch stage (C4): run k ADMM
iterations on the device, rebuild iteration k+1's branch batch (warm start x,
current parameter rows) and solve it once with per-problem timing."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_14995_b200 import ProblemBatch, Solver, synth  # noqa: E402
from paper_2106_14995_b200 import admm as A  # noqa: E402

g = synth.grid(13659, 20467, 4092)
a = A.AdmmSolver(g)
for k in (3, 10, 30):
    while len(a.history) < k:
        a.step()
    x = a.get(A.BRANCH_X)
    prm = a.get(A.BRANCH_PARAMS)
    lo = np.stack([g.bus_vmin[g.br_from], g.bus_vmin[g.br_to], np.full(g.n_branch, -2 * np.pi),
                   np.full(g.n_branch, -2 * np.pi)], 1)
    up = np.stack([g.bus_vmax[g.br_from], g.bus_vmax[g.br_to], np.full(g.n_branch, 2 * np.pi),
                   np.full(g.n_branch, 2 * np.pi)], 1)
    dev = torch.device("cuda", 0)
    t = lambda v: torch.from_numpy(np.ascontiguousarray(v)).to(dev)  # noqa: E731
    b = ProblemBatch(3, 4, t(lo), t(up), t(prm), t(x))
    s = Solver((0,))
    out = Solver.alloc_result(g.n_branch, 4, device=True)
    for _ in range(3):
        s.solve_batch(b, out=out)
    wt = out.per_problem_time.cpu().numpy() * 1e3
    it = out.iterations.cpu().numpy()
    print(f"after ADMM iteration {k}: kernel {out.kernel_time*1e3:.3f} ms; per-branch ms mean {wt.mean():.4f} "
          f"p50 {np.median(wt):.4f} p99 {np.percentile(wt, 99):.4f} max {wt.max():.4f}; iterations mean "
          f"{it.mean():.2f} max {it.max()}; busy warps {wt.sum()/(out.kernel_time*1e3):.0f}", flush=True)
