"""Per-problem latency of the thread vs warp form (per_problem_time field), C1 ncvx d=4 x1,024:
which problems set the launch time.  python scripts/thread_latency.py [fam n d]"""
import os, subprocess, sys

fam, n, d = (sys.argv[1], int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else ("ncvx", 1024, 4)
CODE = r"""
import os, sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2106_14995_b200 import KernelForm, ProblemBatch, Solver, synth
fam, n, d = os.environ['TL_FAM'], int(os.environ['TL_N']), int(os.environ['TL_D'])
b = synth.make(fam, n, d)
dev = torch.device('cuda', 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
db = ProblemBatch(b.family, d, t(b.lower), t(b.upper), t(b.params), t(b.x0))
s = Solver((0,), form=KernelForm[os.environ['TL_FORM']])
out = Solver.alloc_result(n, d, device=True); out.flops = None
for _ in range(3):
    s.solve_batch(db, out=out)
wt = out.per_problem_time.cpu().numpy(); it = out.iterations.cpu().numpy(); cg = out.cg_iterations.cpu().numpy()
o = np.argsort(-wt)[:5]
print(f"{os.environ['TL_LABEL']}: kernel {out.kernel_time*1e3:.3f} ms; per-problem mean {wt.mean()*1e6:.1f} us, "
      f"p99 {np.percentile(wt, 99)*1e6:.1f} us, max {wt.max()*1e6:.1f} us; iterations mean {it.mean():.2f} max {it.max()}")
print("   slowest:", [(int(i), round(wt[i]*1e6, 1), int(it[i]), int(cg[i])) for i in o])
"""
for label, env in (("warp", {"TL_FORM": "WARP"}), ("thread", {"TL_FORM": "THREAD"})):
    e = dict(os.environ, TL_FAM=fam, TL_N=str(n), TL_D=str(d), TL_LABEL=label, **env)
    p = subprocess.run([sys.executable, "-c", CODE], env=e, capture_output=True, text=True)
    print(p.stdout.strip() or p.stderr[-1500:], flush=True)
