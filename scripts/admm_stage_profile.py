"""Per-branch profile of the ADMM branch stage after warm-up: snapshot the C4
(or C5) branch batch after K iterations and solve it once, device-resident,
with per-problem device times and iteration counts (which branches set the
stage time).  python scripts/admm_stage_profile.py [C4|C5] [K]"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_14995_b200 import KernelForm, ProblemBatch, Solver, synth  # noqa: E402
from paper_2106_14995_b200 import admm as A  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "C4"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
if which == "C4":
    g = synth.grid(13659, 20467, 4092)
else:
    nb = int(round(70000 * 13659 / 20467))
    g = synth.grid(nb, 70000, int(0.3 * nb))
run = A.AdmmSolver(g)
for _ in range(K):
    run.step()
n = g.n_branch
lo = np.stack([g.bus_vmin[g.br_from], g.bus_vmin[g.br_to], np.full(n, -2 * np.pi), np.full(n, -2 * np.pi)], 1)
up = np.stack([g.bus_vmax[g.br_from], g.bus_vmax[g.br_to], np.full(n, 2 * np.pi), np.full(n, 2 * np.pi)], 1)
dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
b = ProblemBatch(3, 4, t(lo), t(up), t(run.get(A.BRANCH_PARAMS)), t(run.get(A.BRANCH_X)))
for form in ("THREAD", "WARP"):
    s = Solver((0,), form=KernelForm[form])
    out = Solver.alloc_result(n, 4, device=True)
    s.solve_batch(b, out=out)
    s.solve_batch(b, out=out)
    it = out.iterations.cpu().numpy()
    wt = out.per_problem_time.cpu().numpy()
    st = out.status.cpu().numpy()
    cg = out.cg_iterations.cpu().numpy()
    order = np.argsort(-wt)
    print(f"{which} after {K} iterations, {form} form: kernel {out.kernel_time*1e3:.3f} ms; iterations mean "
          f"{it.mean():.2f} p99 {np.percentile(it, 99):.0f} max {it.max()}; status counts {np.bincount(st)}")
    for i in order[:8]:
        print(f"   branch {i}: {wt[i]*1e3:.3f} ms, {it[i]} iterations, {cg[i]} CG, status {st[i]}, "
              f"{wt[i]/max(it[i],1)*1e6:.2f} us/iteration")
    s.close()

# the long branches alone (what a thread -> warp handoff would leave to a second launch)
s = Solver((0,), form=KernelForm.THREAD)
out = Solver.alloc_result(n, 4, device=True)
s.solve_batch(b, out=out)
it = out.iterations.cpu().numpy()
s.close()
for cut in (16, 32, 64):
    idx = np.nonzero(it > cut)[0]
    if len(idx) == 0:
        continue
    ti = torch.from_numpy(idx).to(dev)
    sb = ProblemBatch(3, 4, b.lower[ti].contiguous(), b.upper[ti].contiguous(), b.params[ti].contiguous(),
                      b.x0[ti].contiguous())
    for form in ("THREAD", "WARP"):
        s = Solver((0,), form=KernelForm[form])
        o = Solver.alloc_result(len(idx), 4, device=True)
        ts = []
        for _ in range(5):
            s.solve_batch(sb, out=o)
            ts.append(o.kernel_time)
        print(f"  {len(idx)} branches with > {cut} iterations alone, {form}: {sorted(ts)[2]*1e3:.3f} ms "
              f"(max iterations {o.iterations.cpu().numpy().max()})")
        s.close()
