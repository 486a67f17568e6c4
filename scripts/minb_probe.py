"""Device-resident median kernel time of several shapes (for library variants)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_14995_b200 import ProblemBatch, Solver, synth  # noqa: E402

s = Solver((0,))
dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
res = []
for fam, n, d in (("branch", 65536, 6), ("branch", 20467, 4), ("ncvx", 32768, 4), ("ncvx", 32768, 8), ("ncvx", 32768, 16)):
    b = synth.make(fam, n, d)
    db = ProblemBatch(b.family, d, t(b.lower), t(b.upper), t(b.params), t(b.x0))
    out = Solver.alloc_result(n, d, device=True)
    ks = []
    for k in range(7):
        s.solve_batch(db, out=out)
        if k >= 2:
            ks.append(out.kernel_time)
    res.append(f"{fam}{d}x{n} {1e3 * sorted(ks)[2]:.3f}")
print(os.environ.get("TB_LIB_PATH", "default").split("/")[-1], " | ".join(res), flush=True)
