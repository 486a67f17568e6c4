"""ADMM iteration rate on C4 (device-timed, CUDA events): python scripts/admm_rate.py [iters]
(TB_LIB_PATH selects a library variant)."""
import os, sys
sys.path.insert(0, ".")
import torch
from paper_2106_14995_b200 import synth
from paper_2106_14995_b200 import admm as A

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
g = synth.grid(13659, 20467, 4092)
opts = A.AdmmOptions(line_limits=os.environ.get("LL", "0") == "1")
a = A.AdmmSolver(g, opts)
for _ in range(5):
    a.step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    a.step()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print(f"{os.path.basename(os.environ.get('TB_LIB_PATH', 'default'))}: {ms:.3f} ms/iter = {1e3 / ms:.1f} iter/s"
      f" (line_limits={opts.line_limits})")
