"""Cycles per TRON iteration of the slow C2 problems vs concurrent warps per SM
(same code, same problems): TB_LIB_PATH=scratch_libs/libtb_phases.so
python scripts/concurrency_probe.py"""
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
lib = _lib.load()
rd = lib.tb_debug_read_phases_branch
buf = (C.c_ulonglong * 16)()
for per_sm in (1, 2, 4, 8, 12, 16):
    n = 148 * per_sm
    idx = np.resize(slow, n)
    sb = ProblemBatch(b.family, 6, b.lower[idx], b.upper[idx], b.params[idx], b.x0[idx])
    s.solve_batch(sb)
    rd(buf)
    rr = s.solve_batch(sb)
    rd(buf)
    ph = np.array(list(buf), dtype=np.float64)
    its = float(np.sum(rr.iterations))
    print(f"{per_sm:2d} warps/SM: kernel {rr.kernel_time*1e3:8.3f} ms, cycles per iteration per warp {ph[7]/its:9,.0f}, "
          f"SM throughput {its / rr.kernel_time / 148 / 1e3:8.1f} k iterations/s/SM", flush=True)
