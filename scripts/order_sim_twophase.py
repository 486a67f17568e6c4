"""List-scheduling simulation of a two-phase ncvx solve with a late cut (K = p50 / p75 / p90 of the
executed iterations; survivors resumed in a second launch): python scripts/order_sim_twophase.py"""
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
    cost = r.flops.astype(float) + 2000.0*r.executed
    idx = makespan(cost, slots); perf = makespan(np.sort(cost)[::-1], slots)
    print(f"d={d}: index {idx:.3g} perfect {perf:.3g} ({perf/idx:.2f}); iterations p50 {np.median(r.executed)} p75 {np.percentile(r.executed,75)} p90 {np.percentile(r.executed,90)}")
    for K in (int(np.percentile(r.executed,50)), int(np.percentile(r.executed,75)), int(np.percentile(r.executed,90))):
        rk = po.solve_batch(b, cfg=TronConfig(max_iter=K), impl='oracle', workers=8)
        c1 = rk.flops.astype(float) + 2000.0*rk.executed
        surv = r.executed > K
        c2 = np.maximum(cost - c1, 0)[surv] + 1500.0
        p1 = makespan(c1, slots)
        p2r = makespan(c2[np.argsort(-rk.pg_norm[surv])], slots)
        p2s = makespan(np.sort(c2)[::-1], slots)
        print(f"   K={K}: survivors {surv.sum()}; phase1 {p1:.3g} + phase2 (pg@K ranked) {p2r:.3g} = {(p1+p2r)/idx:.2f} of index; with a perfect phase-2 order {(p1+p2s)/idx:.2f}")
