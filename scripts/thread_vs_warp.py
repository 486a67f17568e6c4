"""Branch family: warp-per-problem vs thread-per-problem (VT_FORM=WARP / THREAD selects the KernelForm), device-resident
timing and bitwise comparison of every SolveReport field.
python scripts/thread_vs_warp.py [n [fam,fam [variant,variant]]]"""
import os, subprocess, sys

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
CODE = r"""
import os, sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2106_14995_b200 import KernelForm, ProblemBatch, Solver, synth
fam, n = os.environ['VT_FAM'], int(os.environ['VT_N'])
name = fam.rstrip('0123456789'); dim = int(fam[len(name):])
b = synth.make(name, n, dim)
dev = torch.device('cuda', 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
db = ProblemBatch(b.family, dim, t(b.lower), t(b.upper), t(b.params), t(b.x0))
s = Solver((0,), form=KernelForm[os.environ.get('VT_FORM', 'AUTO')])
out = Solver.alloc_result(n, dim, device=True); out.flops = None
s.solve_batch(db, out=out)
ts = []
for _ in range(7):
    s.solve_batch(db, out=out); ts.append(out.kernel_time)
ts.sort()
np.savez('/tmp/tvw_%s_%s.npz' % (fam, os.environ.get('VT_FORM', 'AUTO')),
         **{k: getattr(out, k).cpu().numpy() for k in ('x_star', 'f_star', 'pg_norm', 'status', 'iterations', 'cg_iterations', 'f_evals')})
print(f"form={os.environ.get("VT_FORM")} {fam} x{n}: best {ts[0]*1e3:.3f} ms  median {ts[3]*1e3:.3f} ms")
"""
import numpy as np
fams = sys.argv[2].split(",") if len(sys.argv) > 2 else ["branch6", "branch4"]
variants = sys.argv[3].split(",") if len(sys.argv) > 3 else ["WARP", "THREAD"]
for fam in fams:
    for thr in variants:
        env = dict(os.environ, VT_FAM=fam, VT_N=str(n), VT_FORM=thr)
        p = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
        print(p.stdout.strip() or p.stderr[-1500:], flush=True)
    try:
        a = np.load(f"/tmp/tvw_{fam}_{variants[0]}.npz")
        for thr in variants[1:]:
            b = np.load(f"/tmp/tvw_{fam}_{thr}.npz")
            bad = [k for k in a.files if a[k].tobytes() != b[k].tobytes()]
            print(fam, thr, "bitwise identical" if not bad else f"DIFFER in {bad}", flush=True)
    except Exception as e:
        print(fam, "compare failed", e)
