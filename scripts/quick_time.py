"""Quick host-buffer timing of a few shapes with flop counts (solves/s and TFLOP/s per shape)."""
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
from paper_2106_14995_b200 import Solver, TronConfig, synth
s = Solver((0,))
for name, b in [("branch6", synth.branch(65536, 6)), ("ncvx4", synth.ncvx(65536, 4, 1)), ("ncvx16", synth.ncvx(32768, 16, 19)), ("ncvx32", synth.ncvx(32768, 32, 35))]:
    r = s.solve_batch(b, count_flops=True)
    fl = np.sum(r.flops)
    ts = []
    for _ in range(3):
        r = s.solve_batch(b); ts.append(r.kernel_time)
    kt = min(ts)
    print(f"{name}: kernel {kt*1e3:.2f} ms -> {b.count/kt/1e6:.2f} M solves/s; e2e wall {r.batch_wall_time*1e3:.2f} ms; flops/solve {fl/b.count:.0f} -> {fl/kt/1e12:.3f} TFLOP/s; status {np.bincount(r.status)}", flush=True)
