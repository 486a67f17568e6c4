"""Run-to-run spread of kernel time per launch order (25 launches)."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2106_14995_b200 import KernelForm, LaunchOrder, ProblemBatch, Solver, synth
dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
for fam, n, dim in (("branch", 65536, 6), ("ncvx", 32768, 16), ("ncvx", 32768, 8), ("ncvx", 8192, 32), ("branch", 20467, 4)):
    b = synth.make(fam, n, dim)
    db = ProblemBatch(b.family, dim, t(b.lower), t(b.upper), t(b.params), t(b.x0))
    for order in (LaunchOrder.INDEX, LaunchOrder.START_PG):
        s = Solver((0,), order=order)
        out = Solver.alloc_result(n, dim, device=True)
        ks = []
        for _ in range(25):
            s.solve_batch(db, out=out); ks.append(out.kernel_time * 1e3)
        ks = np.array(ks[1:])
        print(f"{fam}{dim} {order.name}: min {ks.min():.3f} p25 {np.percentile(ks,25):.3f} med {np.median(ks):.3f} p75 {np.percentile(ks,75):.3f} max {ks.max():.3f}", flush=True)
        s.close()
