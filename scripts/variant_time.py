"""Time a workload on each library variant (TB_LIB_PATH), device-resident inputs
(host-buffer timings include the copy pipeline and mislead kernel comparisons):
python scripts/variant_time.py [--fam branch6 --n 65536] lib1.so lib2.so ..."""
import os, subprocess, sys

args = sys.argv[1:]
fam, n = "branch6", 65536
if args and args[0] == "--fam":
    fam, n, args = args[1], int(args[3]), args[4:]
CODE = r"""
import os, sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2106_14995_b200 import ProblemBatch, Solver, synth
fam, n = os.environ['VT_FAM'], int(os.environ['VT_N'])
name = fam.rstrip('0123456789'); dim = int(fam[len(name):])
b = synth.make(name, n, dim)
dev = torch.device('cuda', 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
db = ProblemBatch(b.family, dim, t(b.lower), t(b.upper), t(b.params), t(b.x0))  # device-resident: kernel time only
s = Solver((0,))
out = Solver.alloc_result(n, dim, device=True)
s.solve_batch(db, out=out)
ts = []
for _ in range(5):
    s.solve_batch(db, out=out); ts.append(out.kernel_time)
ts.sort()
print(f"{os.environ['VT_LABEL']:28s} {fam} x{n}: best {ts[0]*1e3:.3f} ms  median {ts[2]*1e3:.3f} ms")
"""
for lib in args:
    env = dict(os.environ, TB_LIB_PATH=lib, VT_FAM=fam, VT_N=str(n), VT_LABEL=os.path.basename(lib))
    p = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    print(p.stdout.strip() or p.stderr[-800:], flush=True)
