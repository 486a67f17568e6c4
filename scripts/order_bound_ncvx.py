"""Perfect-knowledge launch order (oracle flop counts, descending; CALLER
order = one launch) vs index order for ncvx batches: is there a tail left
for a better predictor?  python scripts/order_bound_ncvx.py"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_14995_b200 import LaunchOrder, ProblemBatch, Solver, synth  # noqa: E402

dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
for d, n in [(int(a.split(":")[0]), int(a.split(":")[1])) for a in (sys.argv[1:] or ["8:32768", "16:32768", "64:4096", "128:1024"])]:
    b = synth.ncvx(n, d)
    perm = np.load(f"scratch_libs/perm_ncvx{d}_flops.npy")
    for name, p, order in (("index", np.arange(n), LaunchOrder.INDEX), ("oracle-sorted", perm, LaunchOrder.CALLER),
                           ("start-pg ranked", np.arange(n), LaunchOrder.START_PG)):
        s = Solver((0,), order=order)
        db = ProblemBatch(b.family, d, t(b.lower[p]), t(b.upper[p]), t(b.params[p]), t(b.x0[p]))
        out = Solver.alloc_result(n, d, device=True)
        s.solve_batch(db, out=out)
        ks = []
        for _ in range(5):
            s.solve_batch(db, out=out)
            ks.append(out.kernel_time * 1e3)
        print(f"ncvx{d} x{n} {name:16s}: median {np.median(ks):.3f} ms", flush=True)
        s.close()
