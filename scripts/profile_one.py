"""Run a few solves of one family/size (for ncu captures): python scripts/profile_one.py branch6 8192 [reps]"""
import sys
sys.path.insert(0, ".")
from paper_2106_14995_b200 import Solver, synth

fam, n = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
name = fam.rstrip("0123456789")
dim = int(fam[len(name):]) if fam[len(name):] else 6
b = synth.make(name, n, dim)
s = Solver((0,))
for _ in range(reps):
    r = s.solve_batch(b)
print(f"{fam} x{n}: kernel {r.kernel_time*1e3:.3f} ms")
