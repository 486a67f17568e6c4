"""Quick C3 timing: device kernel time of the ncvx sweep (no parity)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_14995_b200 import ProblemBatch, Solver, synth  # noqa: E402

dims = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else "4,8,16,32,64,128".split(","))]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
s = Solver((0,))
dev = torch.device("cuda", 0)
for d in dims:
    b = synth.ncvx(B, d, seed=3 + d)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    db = ProblemBatch(b.family, d, t(b.lower), t(b.upper), t(b.params), t(b.x0))
    r = s.solve_batch(db)
    ts = []
    for _ in range(2):
        r = s.solve_batch(db)
        ts.append(r.kernel_time)
    it = r.iterations.float().mean().item() if hasattr(r.iterations, "float") else float(np.mean(r.iterations))
    print(f"d={d:4d} B={B} kernel {min(ts)*1e3:9.2f} ms  {B/min(ts):12.0f} solves/s  mean its {it:.2f}", flush=True)
