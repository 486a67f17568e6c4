"""Device-resident A/B of the kernel forms (KernelForm) on the same batches,
with a bitwise cross-check of every SolveReport field between forms:
python scripts/form_time.py [fam:n,fam:n ...] [FORM,FORM ...]
e.g. python scripts/form_time.py branch6:65536,ncvx8:32768 WARP,GROUP"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_14995_b200 import KernelForm, ProblemBatch, Solver, synth  # noqa: E402

work = (sys.argv[1] if len(sys.argv) > 1 else "branch6:65536,branch4:20467,ncvx4:1024,ncvx8:32768").split(",")
forms = (sys.argv[2] if len(sys.argv) > 2 else "WARP,GROUP").split(",")
reps = int(os.environ.get("FT_REPS", 7))
dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
FIELDS = ("x_star", "f_star", "pg_norm", "status", "iterations", "cg_iterations", "f_evals")
s = Solver((0,))
for w in work:
    fam, n = w.split(":")
    n = int(n)
    name = fam.rstrip("0123456789")
    dim = int(fam[len(name):])
    b = synth.make(name, n, dim)
    db = ProblemBatch(b.family, dim, t(b.lower), t(b.upper), t(b.params) if b.params is not None else None, t(b.x0))
    base = None
    for f in forms:
        s.set_form(KernelForm[f])
        out = Solver.alloc_result(n, dim, device=True)
        s.solve_batch(db, out=out)
        ts = []
        for _ in range(reps):
            s.solve_batch(db, out=out)
            ts.append(out.kernel_time)
        ts.sort()
        res = {k: getattr(out, k).cpu().numpy() for k in FIELDS}
        same = ""
        if base is None:
            base = res
        else:
            bad = [k for k in FIELDS if res[k].tobytes() != base[k].tobytes()]
            same = "bitwise = " + forms[0] if not bad else f"DIFFERS from {forms[0]} in {bad}"
        med = ts[len(ts) // 2]
        print(f"{fam:8s} x{n:6d} {f:6s}: best {ts[0]*1e3:8.3f} ms  median {med*1e3:8.3f} ms  "
              f"{n/med/1e6:7.2f} M solves/s  {same}", flush=True)
s.close()
