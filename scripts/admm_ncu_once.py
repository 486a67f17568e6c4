"""22 C4 ADMM iterations (for an ncu capture of the late branch stage: -k regex:admm_gen_branch -s 20 -c 1)."""
import sys; sys.path.insert(0, '.')
from paper_2106_14995_b200 import synth
from paper_2106_14995_b200 import admm as A
g = synth.grid(13659, 20467, 4092)
a = A.AdmmSolver(g)
for _ in range(22):
    a.step()
print("done")
