"""Where the host-buffer (e2e) path spends its time on C2: Python wall, the C
call's wall (batch_wall_time) and the device span of the partition."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_14995_b200 import ProblemBatch, Solver, synth  # noqa: E402

b = synth.branch(65536, 6, seed=2)


def pinned(a):
    p = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    p.copy_(torch.from_numpy(np.ascontiguousarray(a)))
    return p.numpy()


hb = ProblemBatch(b.family, 6, pinned(b.lower), pinned(b.upper), pinned(b.params), pinned(b.x0))
s = Solver((0,))
out = Solver.alloc_result(65536, 6)
tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64}
for name in ("x_star", "f_star", "pg_norm", "status", "iterations", "cg_iterations", "f_evals", "per_problem_time"):
    a = getattr(out, name)
    setattr(out, name, torch.empty(a.shape, dtype=tdt[a.dtype], pin_memory=True).numpy())
for _ in range(3):
    s.solve_batch(hb, out=out)
rows = []
for _ in range(10):
    t0 = time.perf_counter()
    s.solve_batch(hb, out=out)
    rows.append((time.perf_counter() - t0, out.batch_wall_time, out.partition_times[0], out.kernel_time))
r = np.median(np.array(rows), axis=0) * 1e3
print(f"python wall {r[0]:.3f} ms | C wall {r[1]:.3f} ms | device partition span {r[2]:.3f} ms | "
      f"first kernel start..last D2H {r[3]:.3f} ms")
