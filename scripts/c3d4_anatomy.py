"""C3 d=4 (32,768 ncvx, thread form) anatomy: the slowest problems' device
time and iterations in the batch vs the same problems alone.
python scripts/c3d4_anatomy.py"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_14995_b200 import KernelForm, ProblemBatch, Solver, synth  # noqa: E402

dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
b = synth.ncvx(32768, 4)
db = ProblemBatch(b.family, 4, t(b.lower), t(b.upper), t(b.params), t(b.x0))
s = Solver((0,), form=KernelForm.THREAD)
out = Solver.alloc_result(32768, 4, device=True)
ks = []
for _ in range(7):
    s.solve_batch(db, out=out)
    ks.append(out.kernel_time)
wt = out.per_problem_time.cpu().numpy()
it = out.iterations.cpu().numpy()
cg = out.cg_iterations.cpu().numpy()
print(f"kernel median {np.median(ks)*1e3:.3f} ms; per-problem time p50 {np.median(wt)*1e6:.1f} us p99 "
      f"{np.percentile(wt, 99)*1e6:.1f} max {wt.max()*1e6:.1f}; iterations p50 {np.median(it)} p99 "
      f"{np.percentile(it, 99)} max {it.max()}")
order = np.argsort(-wt)[:6]
for i in order:
    w = i // 32
    sib = it[w * 32:(w + 1) * 32]
    print(f"  problem {i}: {wt[i]*1e6:.1f} us, {it[i]} it, {cg[i]} cg; warp {w}: sibling iterations max {sib.max()} "
          f"mean {sib.mean():.1f}")
i = int(order[0])
for form in ("THREAD", "WARP"):
    s2 = Solver((0,), form=KernelForm[form])
    sb = ProblemBatch(b.family, 4, db.lower[i:i + 1], db.upper[i:i + 1], db.params[i:i + 1], db.x0[i:i + 1])
    o = Solver.alloc_result(1, 4, device=True)
    for _ in range(5):
        s2.solve_batch(sb, out=o)
    print(f"  slowest problem alone, {form}: {o.per_problem_time.cpu().numpy()[0]*1e6:.1f} us")
    s2.close()
# the longest-iteration problem
j = int(np.argmax(it))
print(f"  most iterations: problem {j}: {it[j]} it, {wt[j]*1e6:.1f} us in the batch")
