"""Per-problem latency distribution of one C2 launch (device-resident inputs):
how much of the kernel is the tail of long-running problems."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_14995_b200 import ProblemBatch, Solver, synth  # noqa: E402

fam = sys.argv[1] if len(sys.argv) > 1 else "branch6"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
name = fam.rstrip("0123456789")
d = int(fam[len(name):])
b = synth.make(name, N, d)
dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
db = ProblemBatch(b.family, d, t(b.lower), t(b.upper), t(b.params), t(b.x0))
s = Solver((0,))
out = Solver.alloc_result(N, d, device=True)
for _ in range(3):
    s.solve_batch(db, out=out)
wt = out.per_problem_time.cpu().numpy() * 1e3
it = out.iterations.cpu().numpy()
st = out.status.cpu().numpy()
print(f"{fam} x{N}: kernel {out.kernel_time*1e3:.3f} ms; per-problem ms: mean {wt.mean():.4f} p50 {np.median(wt):.4f} "
      f"p99 {np.percentile(wt, 99):.4f} p99.9 {np.percentile(wt, 99.9):.4f} max {wt.max():.4f}")
print(f"  sum of per-problem time / kernel = {wt.sum() / (out.kernel_time*1e3):.0f} concurrent warps on average")
order = np.argsort(-wt)[:10]
for i in order:
    print(f"  problem {i}: {wt[i]:.3f} ms, iterations {it[i]}, status {st[i]}")
for thr in (0.05, 0.1, 0.2, 0.5, 1.0):
    m = wt > thr
    print(f"  problems > {thr} ms: {m.sum()} ({100*m.mean():.2f}%), their time share {100*wt[m].sum()/wt.sum():.1f}%")
