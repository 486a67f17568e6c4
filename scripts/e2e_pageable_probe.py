"""C2 end to end through the public API with PAGEABLE numpy buffers (the
library's pinned staging): median wall per call, for a launch order."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2106_14995_b200 import LaunchOrder, Solver, synth  # noqa: E402

b = synth.branch(65536, 6, seed=2)
for order in (LaunchOrder.AUTO, LaunchOrder.INDEX):
    s = Solver((0,), order=order)
    out = Solver.alloc_result(65536, 6)
    for _ in range(3):
        s.solve_batch(b, out=out)
    ts = []
    for _ in range(11):
        t0 = time.perf_counter()
        s.solve_batch(b, out=out)
        ts.append(time.perf_counter() - t0)
    ms = float(np.median(ts)) * 1e3
    print(f"pageable {order.name}: {ms:.3f} ms = {65536 / ms / 1e3:.2f} M solves/s; kernel {out.kernel_time*1e3:.3f} ms")
    s.close()
