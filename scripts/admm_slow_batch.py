"""The genuinely slow ADMM branch solves (C4 after 30 iterations), replicated
4 per SM, solved twice (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2106_14995_b200 import ProblemBatch, Solver, synth  # noqa: E402
from paper_2106_14995_b200 import admm as A  # noqa: E402

g = synth.grid(13659, 20467, 4092)
a = A.AdmmSolver(g)
for _ in range(30):
    a.step()
x, prm = a.get(A.BRANCH_X), a.get(A.BRANCH_PARAMS)
lo = np.stack([g.bus_vmin[g.br_from], g.bus_vmin[g.br_to], np.full(g.n_branch, -2 * np.pi),
               np.full(g.n_branch, -2 * np.pi)], 1)
up = np.stack([g.bus_vmax[g.br_from], g.bus_vmax[g.br_to], np.full(g.n_branch, 2 * np.pi),
               np.full(g.n_branch, 2 * np.pi)], 1)
s = Solver((0,))
r = s.solve_batch(ProblemBatch(3, 4, lo, up, prm, x))
wt0 = np.asarray(r.per_problem_time)
slow = np.nonzero(wt0 > 0.5 * wt0.max())[0]
idx = np.resize(slow, 148 * 4)
sb = ProblemBatch(3, 4, lo[idx], up[idx], prm[idx], x[idx])
for _ in range(2):
    rr = s.solve_batch(sb)
print(len(slow), rr.kernel_time)
