"""One solve per C3 dimension (for an ncu metric pass over the sweep)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_14995_b200 import ProblemBatch, Solver, synth  # noqa: E402

s = Solver((0,))
dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
for d, B in ((4, 32768), (8, 32768), (16, 32768), (32, 8192), (64, 4096), (128, 1024)):
    b = synth.ncvx(B, d, seed=3 + d)
    db = ProblemBatch(b.family, d, t(b.lower), t(b.upper), t(b.params), t(b.x0))
    out = Solver.alloc_result(B, d, device=True)
    s.solve_batch(db, out=out)
    print(d, B, out.kernel_time, flush=True)
