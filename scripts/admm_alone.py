"""The C4 branch-stage batch after 30 ADMM iterations, solved alone (device-resident) for timing /
captures of the stage without the rest of the iteration."""
import os, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2106_14995_b200 import ProblemBatch, Solver, synth
from paper_2106_14995_b200 import admm as A
g = synth.grid(13659, 20467, 4092)
a = A.AdmmSolver(g)
for _ in range(30): a.step()
x = a.get(A.BRANCH_X); prm = a.get(A.BRANCH_PARAMS)
lo = np.stack([g.bus_vmin[g.br_from], g.bus_vmin[g.br_to], np.full(g.n_branch, -2*np.pi), np.full(g.n_branch, -2*np.pi)], 1)
up = np.stack([g.bus_vmax[g.br_from], g.bus_vmax[g.br_to], np.full(g.n_branch, 2*np.pi), np.full(g.n_branch, 2*np.pi)], 1)
dev = torch.device("cuda", 0); t = lambda v: torch.from_numpy(np.ascontiguousarray(v)).to(dev)
s = Solver((0,))
b = ProblemBatch(3, 4, t(lo), t(up), t(prm), t(x)); out = Solver.alloc_result(g.n_branch, 4, device=True)
for _ in range(3): s.solve_batch(b, out=out)
wt = out.per_problem_time.cpu().numpy(); it = out.iterations.cpu().numpy(); cg = out.cg_iterations.cpu().numpy()
order = np.argsort(-wt)[:5]
print("full launch", out.kernel_time*1e3, "ms")
for i in order:
    b1 = ProblemBatch(3, 4, t(lo[i:i+1]), t(up[i:i+1]), t(prm[i:i+1]), t(x[i:i+1])); o1 = Solver.alloc_result(1, 4, device=True)
    for _ in range(3): s.solve_batch(b1, out=o1)
    print(f"branch {i}: in-batch {wt[i]*1e3:.3f} ms, alone {o1.per_problem_time.cpu().numpy()[0]*1e3:.3f} ms, iterations {it[i]}, cg {cg[i]}")
