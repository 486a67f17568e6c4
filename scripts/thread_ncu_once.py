"""One C3 ncvx d=4 x 32,768 solve (thread-per-problem form) for an ncu capture:
ncu --set full -k regex:tron_thread_kernel -c 1 python scripts/thread_ncu_once.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_14995_b200 import ProblemBatch, Solver, synth  # noqa: E402

s = Solver((0,))
dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
fam, d, B = (sys.argv[1], int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else ("ncvx", 4, 32768)
b = synth.make(fam, B, d)
db = ProblemBatch(b.family, d, t(b.lower), t(b.upper), t(b.params), t(b.x0))
out = Solver.alloc_result(B, d, device=True)
s.solve_batch(db, out=out)
print(fam, d, B, out.kernel_time, flush=True)
