"""Phase profile of the slow (>= 150-iteration) C2 problems only:
TB_LIB_PATH=scratch_libs/libtb_phases.so python scripts/phase_slow.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2106_14995_b200 import ProblemBatch, Solver, _lib, synth  # noqa: E402

b = synth.branch(65536, 6, seed=2)
s = Solver((0,))
r = s.solve_batch(b)
slow = np.nonzero(np.asarray(r.iterations) >= 150)[0]
reps = max(1, 8192 // len(slow))
idx = np.tile(slow, reps)
sb = ProblemBatch(b.family, 6, b.lower[idx], b.upper[idx], b.params[idx], b.x0[idx])
lib = _lib.load()
rd = lib.tb_debug_read_phases_branch
buf = (C.c_ulonglong * 16)()
s.solve_batch(sb)
rd(buf)
rr = s.solve_batch(sb)
rd(buf)
ph = np.array(list(buf), dtype=np.float64)
n = len(idx)
its = float(np.sum(rr.iterations))
cg = float(np.sum(rr.cg_iterations))
print(f"{len(slow)} slow problems x{reps}: kernel {rr.kernel_time*1e3:.3f} ms; cycles/solve {ph[7]/n:,.0f}; "
      f"iterations/solve {its/n:.1f} (cg {cg/n:.1f}); cycles per iteration {ph[7]/its:,.0f}")
names = {0: "hessian", 1: "cauchy", 2: "ccf", 3: "pcg", 4: "line_search", 5: "subspace(total)", 6: "f_eval+prepare"}
for k, nm in names.items():
    print(f"  {nm:20s} {100*ph[k]/ph[7]:5.1f}%  {ph[k]/its:9,.0f} cycles/iteration")
