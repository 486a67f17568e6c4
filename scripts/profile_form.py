"""Device-resident solves of one family/size in one kernel form (for ncu
captures): python scripts/profile_form.py branch6 65536 GROUP [reps]"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_14995_b200 import KernelForm, ProblemBatch, Solver, synth  # noqa: E402

fam, n, form = sys.argv[1], int(sys.argv[2]), sys.argv[3]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
name = fam.rstrip("0123456789")
dim = int(fam[len(name):])
b = synth.make(name, n, dim)
dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
db = ProblemBatch(b.family, dim, t(b.lower), t(b.upper), t(b.params) if b.params is not None else None, t(b.x0))
s = Solver((0,), form=KernelForm[form])
out = Solver.alloc_result(n, dim, device=True)
for _ in range(reps):
    s.solve_batch(db, out=out)
print(f"{fam} x{n} {form}: kernel {out.kernel_time*1e3:.3f} ms")
