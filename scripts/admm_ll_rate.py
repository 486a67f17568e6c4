"""ADMM iteration rate with line limits (the fused augmented-Lagrangian
branch stage, dim 6) on C4 and C5 (single process, events around run()):
python scripts/admm_ll_rate.py [iters] (TB_LIB_PATH selects a build)."""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2106_14995_b200 import admm as A  # noqa: E402
from paper_2106_14995_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
nb = int(round(70000 * 13659 / 20467))
for name, g in (("C4", synth.grid(13659, 20467, 4092)), ("C5", synth.grid(nb, 70000, int(0.3 * nb)))):
    a = A.AdmmSolver(g, A.AdmmOptions(line_limits=True))
    a.run(3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    a.run(n)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{os.path.basename(os.environ.get('TB_LIB_PATH', 'default'))} {name} line limits: {ms:.3f} ms/iter = "
          f"{1e3 / ms:.1f} iter/s", flush=True)
    a.close()
