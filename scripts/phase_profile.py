"""Per-phase share of warp time (debug build with -DTB_PHASES):
TB_LIB_PATH=scratch_libs/libtb_phases.so python scripts/phase_profile.py branch6 65536
   [saved.npz: solve that batch (lo, up, prm, x) with the warp form instead]"""
import ctypes as C, os, sys
sys.path.insert(0, ".")
import numpy as np
from paper_2106_14995_b200 import Solver, _lib, synth

fam, n = sys.argv[1], int(sys.argv[2])
name = fam.rstrip("0123456789"); dim = int(fam[len(name):])
name = {"branch": "branch"}.get(name, name)
if len(sys.argv) > 3:  # a saved batch (npz with lo, up, prm, x), e.g. the ADMM stage's long branches
    from paper_2106_14995_b200 import Family, KernelForm, ProblemBatch
    z = np.load(sys.argv[3])
    b = ProblemBatch(int(Family[name.upper()]), dim, z["lo"], z["up"], z["prm"], z["x"])
    n = b.count
    s = Solver((0,), form=KernelForm.WARP)
else:
    b = synth.make(name, n, dim)
    s = Solver((0,))
lib = _lib.load()
rd = getattr(lib, f"tb_debug_read_phases_{name}")
buf = (C.c_ulonglong * 16)()
s.solve_batch(b); rd(buf)
r = s.solve_batch(b); rd(buf)
ph = np.array(list(buf), dtype=np.float64)
names = ["hessian", "cauchy", "ccf", "pcg", "line_search", "subspace(total)", "f_eval", "TOTAL"]
sub_other = ph[5] - ph[2] - ph[3] - ph[4]
rest = ph[7] - ph[0] - ph[1] - ph[5] - ph[6]
tot = ph[7]
its = float(np.sum(r.iterations))
print(f"{fam} x{n}: kernel {r.kernel_time*1e3:.3f} ms; mean warp cycles/solve {tot/n:,.0f}; per executed problem-iteration ~{tot/its:,.0f} (iterations incl. fast-forwarded)")
for k, v in [("hessian", ph[0]), ("cauchy", ph[1]), ("ccf", ph[2]), ("pcg", ph[3]), ("line_search", ph[4]),
             ("subspace other", sub_other), ("f_eval+prepare", ph[6]), ("rest (grad, radius, setup)", rest)]:
    print(f"  {k:28s} {100*v/tot:5.1f}%  {v/n:10,.0f} cycles/solve")
if ph[8] + ph[9] + ph[10] + ph[11] > 0:  # block kernel (d > 32) breakdown
    for k, v in [("  pcg: trsv_fwd (loop)", ph[8]), ("  pcg: trsv_bwd (loop)", ph[9]), ("  pcg: gemv_c", ph[10]),
                 ("  ccf: chol attempts", ph[11])]:
        print(f"  {k:28s} {100*v/tot:5.1f}%  {v/n:10,.0f} cycles/solve")
