"""Host timeline of C2 with pageable buffers: run under a TB_TRACE_HOST build (TB_LIB_PATH=...)
to print the staging / transfer / solve / copy-out marks of tb_solve_batch."""
import sys, time; sys.path.insert(0,'.')
import numpy as np
from paper_2106_14995_b200 import Solver, synth
b = synth.branch(65536, 6, seed=2)
s = Solver((0,))
out = Solver.alloc_result(65536, 6)
for _ in range(4):
    t0=time.perf_counter(); s.solve_batch(b, out=out); print("call %.3f ms kernel %.3f"%((time.perf_counter()-t0)*1e3, out.kernel_time*1e3), file=sys.stderr)
