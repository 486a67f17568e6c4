"""One warp-form launch of C1's slowest problem (94) replicated once per SM:
the lone chain's latency, for an ncu source capture (-k regex:tron_solve -s 2 -c 1)."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_14995_b200 import KernelForm, ProblemBatch, Solver, synth  # noqa: E402

dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
b = synth.ncvx(1024, 4)
n = 148
sb = ProblemBatch(b.family, 4, t(np.repeat(b.lower[94:95], n, 0)), t(np.repeat(b.upper[94:95], n, 0)),
                  t(np.repeat(b.params[94:95], n, 0)), t(np.repeat(b.x0[94:95], n, 0)))
s = Solver((0,), form=KernelForm.WARP)
out = Solver.alloc_result(n, 4, device=True)
for _ in range(4):
    s.solve_batch(sb, out=out)
print(out.kernel_time)
