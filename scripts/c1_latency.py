"""C1 (1,024 ncvx d=4) latency anatomy: kernel time vs the slowest problem's
own device time (globaltimer) and its iteration count.
python scripts/c1_latency.py"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_14995_b200 import KernelForm, ProblemBatch, Solver, synth  # noqa: E402

dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
b = synth.ncvx(1024, 4)
db = ProblemBatch(b.family, 4, t(b.lower), t(b.upper), t(b.params), t(b.x0))
for form in ("AUTO", "WARP", "THREAD"):
    s = Solver((0,), form=KernelForm[form])
    out = Solver.alloc_result(1024, 4, device=True)
    ks = []
    for _ in range(20):
        s.solve_batch(db, out=out)
        ks.append(out.kernel_time)
    wt = out.per_problem_time.cpu().numpy()
    it = out.iterations.cpu().numpy()
    i = int(np.argmax(wt))
    print(f"{form:6s}: kernel median {np.median(ks)*1e6:.1f} us best {min(ks)*1e6:.1f} us; slowest problem {i}: "
          f"{wt[i]*1e6:.1f} us, {it[i]} iterations ({wt[i]/max(it[i],1)*1e6:.2f} us/it); problem 94: "
          f"{wt[94]*1e6:.1f} us / {it[94]} it; per-problem p50 {np.median(wt)*1e6:.1f} us", flush=True)
    s.close()
# a single problem alone (pure latency)
for n in (1, 148, 1024):
    sb = ProblemBatch(b.family, 4, db.lower[94:95].repeat(n, 1), db.upper[94:95].repeat(n, 1),
                      db.params[94:95].repeat(n, 1), db.x0[94:95].repeat(n, 1))
    s = Solver((0,), form=KernelForm.WARP)
    out = Solver.alloc_result(n, 4, device=True)
    ks = []
    for _ in range(20):
        s.solve_batch(sb, out=out)
        ks.append(out.kernel_time)
    wt = out.per_problem_time.cpu().numpy()
    print(f"problem 94 x{n}: kernel median {np.median(ks)*1e6:.1f} us; its own time {wt.max()*1e6:.1f} us", flush=True)
    s.close()
# the thread form on the same lone problem (one thread; 32 identical copies run in lockstep)
for n in (1, 32, 148):
    sb = ProblemBatch(b.family, 4, db.lower[94:95].repeat(n, 1), db.upper[94:95].repeat(n, 1),
                      db.params[94:95].repeat(n, 1), db.x0[94:95].repeat(n, 1))
    s = Solver((0,), form=KernelForm.THREAD)
    out = Solver.alloc_result(n, 4, device=True)
    ks = []
    for _ in range(20):
        s.solve_batch(sb, out=out)
        ks.append(out.kernel_time)
    wt = out.per_problem_time.cpu().numpy()
    print(f"THREAD problem 94 x{n}: kernel median {np.median(ks)*1e6:.1f} us; its own time {wt.max()*1e6:.1f} us",
          flush=True)
    s.close()
