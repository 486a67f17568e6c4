"""Distribution of per-branch device time and executed work for a saved ADMM
stage batch (npz: lo, up, prm, x): which branches set the stage time.
python scripts/stage_long_dist.py saved.npz"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_14995_b200 import KernelForm, ProblemBatch, Solver  # noqa: E402

z = np.load(sys.argv[1])
dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
b = ProblemBatch(3, 4, t(z["lo"]), t(z["up"]), t(z["prm"]), t(z["x"]))
n = b.count
res = {}
for ff in (0, 1, 2):
    for form in ("THREAD", "WARP"):
        s = Solver((0,), form=KernelForm[form], fast_forward=ff)
        out = Solver.alloc_result(n, 4, device=True)
        for _ in range(3):
            s.solve_batch(b, out=out)
        res[(ff, form)] = (out.kernel_time, out.per_problem_time.cpu().numpy().copy(), out.iterations.cpu().numpy().copy())
        s.close()
        print(f"ff={ff} {form}: kernel {out.kernel_time*1e3:.3f} ms; per-branch time p50 "
              f"{np.percentile(res[(ff, form)][1], 50)*1e3:.3f} p90 {np.percentile(res[(ff, form)][1], 90)*1e3:.3f} "
              f"max {res[(ff, form)][1].max()*1e3:.3f} ms", flush=True)
s = Solver((0,), form=KernelForm.WARP, fast_forward=2)
r2 = s.solve_batch(b, count_flops=True)
s.close()
s = Solver((0,), form=KernelForm.WARP, fast_forward=1)
r1 = s.solve_batch(b, count_flops=True)
s.close()
f1, f2 = (np.asarray(r.flops.cpu() if hasattr(r.flops, "cpu") else r.flops, dtype=np.float64) for r in (r1, r2))
it = np.asarray(r1.iterations.cpu() if hasattr(r1.iterations, "cpu") else r1.iterations)
frac = f2 / np.maximum(f1, 1)
wt = res[(1, "THREAD")][1]
order = np.argsort(-wt)
print("executed / credited flops: p10 %.3f p50 %.3f p90 %.3f" % tuple(np.percentile(frac, [10, 50, 90])))
print("slowest (thread form, ff=1): time ms, iterations, executed-iteration estimate (frac * iterations)")
for i in order[:12]:
    print(f"  {i:5d}: {wt[i]*1e3:.3f} ms  {it[i]} it  ~{frac[i]*it[i]:.0f} executed  "
          f"{wt[i]/max(frac[i]*it[i],1)*1e6:.2f} us/executed it")
ex = frac * it
print("executed iterations: p50 %.0f p90 %.0f p99 %.0f max %.0f" % tuple(np.percentile(ex, [50, 90, 99, 100])))
