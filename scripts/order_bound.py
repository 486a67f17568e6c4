"""Upper bound of launch ordering on C2: the batch permuted on the host by a
saved order (e.g. the oracle's executed iteration counts, descending) and
solved in index order, vs the library's own ranking.
python scripts/order_bound.py perm1.npy [perm2.npy ...]"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_14995_b200 import LaunchOrder, ProblemBatch, Solver, synth  # noqa: E402

dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
b = synth.branch(65536, 6)
cases = [("library ranking", np.arange(65536), LaunchOrder.AUTO)]
cases += [(f"host perm {p}, one launch (CALLER)", np.load(p), LaunchOrder.CALLER) for p in sys.argv[1:]]
for r in range(2):
    for name, p, order in cases:
        s = Solver((0,), order=order)
        db = ProblemBatch(b.family, 6, t(b.lower[p]), t(b.upper[p]), t(b.params[p]), t(b.x0[p]))
        out = Solver.alloc_result(65536, 6, device=True)
        s.solve_batch(db, out=out)
        ks = []
        for _ in range(9):
            s.solve_batch(db, out=out)
            ks.append(out.kernel_time * 1e3)
        print(f"{name:60s}: median {np.median(ks):.3f} ms", flush=True)
        s.close()
