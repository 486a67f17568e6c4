"""Phase profile of the slowest ADMM branch solves (C4, after 30 iterations),
replicated to fill the GPU: TB_LIB_PATH=scratch_libs/libtb_phases.so python scripts/admm_slow_phases.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2106_14995_b200 import ProblemBatch, Solver, _lib, synth  # noqa: E402
from paper_2106_14995_b200 import admm as A  # noqa: E402

g = synth.grid(13659, 20467, 4092)
a = A.AdmmSolver(g)
for _ in range(30):
    a.step()
x, prm = a.get(A.BRANCH_X), a.get(A.BRANCH_PARAMS)
lo = np.stack([g.bus_vmin[g.br_from], g.bus_vmin[g.br_to], np.full(g.n_branch, -2 * np.pi),
               np.full(g.n_branch, -2 * np.pi)], 1)
up = np.stack([g.bus_vmax[g.br_from], g.bus_vmax[g.br_to], np.full(g.n_branch, 2 * np.pi),
               np.full(g.n_branch, 2 * np.pi)], 1)
s = Solver((0,))
r = s.solve_batch(ProblemBatch(3, 4, lo, up, prm, x))
its = np.asarray(r.iterations)
wt0 = np.asarray(r.per_problem_time)
slow = np.nonzero(wt0 > 0.5 * wt0.max())[0]  # genuinely long solves (by wall time, not iteration count)
print(f"{len(slow)} branches slower than half the max ({wt0.max()*1e3:.2f} ms); iterations {its[slow][:8]}, "
      f"cg {np.asarray(r.cg_iterations)[slow][:8]}, f_evals {np.asarray(r.f_evals)[slow][:8]}")
idx = np.resize(slow, 148 * 4)
sb = ProblemBatch(3, 4, lo[idx], up[idx], prm[idx], x[idx])
lib = _lib.load()
rd = lib.tb_debug_read_phases_branch
buf = (C.c_ulonglong * 16)()
s.solve_batch(sb)
rd(buf)
rr = s.solve_batch(sb)
rd(buf)
ph = np.array(list(buf), dtype=np.float64)
it = float(np.sum(rr.iterations))
print(f"kernel {rr.kernel_time*1e3:.3f} ms; cycles per iteration {ph[7]/it:,.0f}")
for k, nm in {0: "hessian", 1: "cauchy", 2: "ccf", 3: "pcg", 4: "line_search", 5: "subspace(total)",
              6: "f_eval+prepare"}.items():
    print(f"  {nm:18s} {100*ph[k]/ph[7]:5.1f}%  {ph[k]/it:8,.0f} cycles/iteration")

# effective SM clock of these solves: clock64 cycles per problem / globaltimer wall
wt = np.asarray(rr.per_problem_time)
print(f"mean clock64 cycles per problem {ph[7]/len(idx):,.0f}; mean wall {wt.mean()*1e3:.3f} ms -> "
      f"effective SM clock {ph[7]/len(idx)/wt.mean()/1e6:,.0f} MHz")
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    print("NVML SM clock now", pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), "MHz; max",
          pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
except Exception as e:
    print("nvml", e)
