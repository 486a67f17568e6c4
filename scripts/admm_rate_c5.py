"""ADMM iteration rate on C4 and C5 (single process, device events around
blocking steps): python scripts/admm_rate_c5.py [iters] (TB_LIB_PATH selects a build)."""
import os, sys
sys.path.insert(0, ".")
import torch
from paper_2106_14995_b200 import synth
from paper_2106_14995_b200 import admm as A

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
nb = int(round(70000 * 13659 / 20467))
for name, g in (("C4", synth.grid(13659, 20467, 4092)), ("C5", synth.grid(nb, 70000, int(0.3 * nb)))):
    a = A.AdmmSolver(g)
    a.run(5)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    a.run(n)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{os.path.basename(os.environ.get('TB_LIB_PATH', 'default'))} {name}: {ms:.3f} ms/iter = {1e3 / ms:.1f} iter/s")
    a.close()
