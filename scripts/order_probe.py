"""Does launch order matter?  C2 (and other batches) device-resident, solved
in the given order vs permuted by a saved order (e.g. descending initial
projected-gradient norm): python scripts/order_probe.py perm.npy"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_14995_b200 import ProblemBatch, Solver, synth  # noqa: E402

dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
b = synth.branch(65536, 6)
perm = np.load(sys.argv[1])
rng = np.random.default_rng(1)
orders = {"given": np.arange(65536), "pg-desc": perm, "pg-asc": perm[::-1].copy(), "random": rng.permutation(65536)}
s = Solver((0,))
res = {}
for r in range(3):
    for name, p in orders.items():
        db = ProblemBatch(b.family, 6, t(b.lower[p]), t(b.upper[p]), t(b.params[p]), t(b.x0[p]))
        out = Solver.alloc_result(65536, 6, device=True)
        ks = []
        for _ in range(9):
            s.solve_batch(db, out=out)
            ks.append(out.kernel_time)
        res.setdefault(name, []).append(np.median(ks) * 1e3)
        if r == 0:
            inv = np.empty_like(p)
            inv[p] = np.arange(65536)
            x = out.x_star.cpu().numpy()[inv]
            res.setdefault("x_" + name, x)
for name in orders:
    print(f"{name:8s}: median kernel ms per round {['%.3f' % v for v in res[name]]}")
for name in orders:
    assert np.array_equal(res["x_" + name].view(np.int64), res["x_given"].view(np.int64)), name
print("x_star identical in every order")
