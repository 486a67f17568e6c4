"""Eight C4 iterations through the sharded driver at world 1 (for an ncu / nsys-style capture of one ADMM
iteration's kernels)."""
import sys, os
sys.path.insert(0, '.')
from paper_2106_14995_b200 import admm as A, synth
g = synth.grid(13659, 20467, 4092)
run = A.ShardedAdmm(g, 0, 1, 0)
for _ in range(8):
    run.step()
