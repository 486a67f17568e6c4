"""Launch order A/B (device-resident, same library): median kernel time of
LaunchOrder.INDEX vs START_PG (and AUTO), interleaved rounds.
python scripts/order_ab.py fam:n[,fam:n...] [form]"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_14995_b200 import KernelForm, LaunchOrder, ProblemBatch, Solver, synth  # noqa: E402

dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
form = KernelForm[sys.argv[2]] if len(sys.argv) > 2 else KernelForm.AUTO
for w in sys.argv[1].split(","):
    fam, n = w.split(":")
    n = int(n)
    name = fam.rstrip("0123456789")
    dim = int(fam[len(name):])
    b = synth.make(name, n, dim)
    db = ProblemBatch(b.family, dim, t(b.lower), t(b.upper), t(b.params) if b.params is not None else None, t(b.x0))
    res = {}
    for r in range(3):
        for order in (LaunchOrder.INDEX, LaunchOrder.START_PG, LaunchOrder.AUTO):
            s = Solver((0,), form=form, order=order)
            out = Solver.alloc_result(n, dim, device=True)
            s.solve_batch(db, out=out)
            ks = []
            for _ in range(9):
                s.solve_batch(db, out=out)
                ks.append(out.kernel_time)
            res.setdefault(order.name, []).append(float(np.median(ks)) * 1e3)
            s.close()
    print(f"{fam:8s} x{n:6d} {form.name:6s}: " + "  ".join(f"{k} {np.median(v):8.3f} ms" for k, v in res.items()),
          flush=True)
