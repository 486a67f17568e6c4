"""List-scheduling simulation of a one-shot launch (slots = resident warps) on oracle cost data: index order vs perfect order vs a two-phase solve (K iterations for all, then the survivors ranked by pg@K).  python scripts/order_sim.py"""
import sys; sys.path.insert(0,'/root/repo')
import numpy as np, heapq
from oracle import pyoracle as po
from paper_2106_14995_b200 import synth, TronConfig
po.set_fast_forward(True)
def makespan(costs, slots):
    h=[0.0]*slots; heapq.heapify(h)
    for c in costs:
        t=heapq.heappop(h); heapq.heappush(h, t+c)
    return max(h)
for d, N, slots in ((8, 32768, 148*28), (16, 32768, 148*20)):
    b = synth.ncvx(N, d)
    r = po.solve_batch(b, impl='oracle', workers=8)
    cost = r.flops.astype(float) + 2000.0*r.executed  # flops + per-iteration overhead proxy
    idx = makespan(cost, slots); perf = makespan(np.sort(cost)[::-1], slots)
    print(f"d={d}: index {idx:.3g}  perfect {perf:.3g}  ratio {perf/idx:.2f}  (lower bound sum/slots {cost.sum()/slots:.3g})")
    for K in (2, 3, 4):
        rk = po.solve_batch(b, cfg=TronConfig(max_iter=K), impl='oracle', workers=8)
        c1 = rk.flops.astype(float) + 2000.0*rk.executed
        surv = (rk.iterations >= K) & (r.iterations > K)
        c2 = np.maximum(cost - c1, 0)[surv] + 1500.0   # remaining + resume overhead (hessian re-eval etc.)
        key = rk.pg_norm[surv]
        p1 = makespan(c1, slots)
        p2 = makespan(c2[np.argsort(-key)], slots)
        p2i = makespan(c2, slots)
        print(f"   K={K}: phase1 {p1:.3g} + phase2 ranked {p2:.3g} = {p1+p2:.3g} (ratio {(p1+p2)/idx:.2f}); phase2 unranked {p2i:.3g}; survivors {surv.sum()}")
