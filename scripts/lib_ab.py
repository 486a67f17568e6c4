"""A/B of library builds on the same device-resident batches (interleaved
rounds, median kernel time): python scripts/lib_ab.py fam:n[,fam:n] lib1.so lib2.so ...
(AB_ORDER=INDEX|START_PG|AUTO sets the launch order where the build has it)"""
import os
import subprocess
import sys

work = sys.argv[1]
libs = sys.argv[2:]
rounds = int(os.environ.get("AB_ROUNDS", 3))
CODE = r"""
import os, sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2106_14995_b200 import ProblemBatch, Solver, synth
dev = torch.device('cuda', 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
s = Solver((0,))
if os.environ.get("AB_ORDER") and hasattr(s._lib, "tb_context_set_order"):
    from paper_2106_14995_b200 import LaunchOrder
    s.set_order(LaunchOrder[os.environ["AB_ORDER"]])
for w in os.environ['AB_WORK'].split(','):
    fam, n = w.split(':'); n = int(n)
    name = fam.rstrip('0123456789'); dim = int(fam[len(name):])
    b = synth.make(name, n, dim)
    db = ProblemBatch(b.family, dim, t(b.lower), t(b.upper), t(b.params) if b.params is not None else None, t(b.x0))
    out = Solver.alloc_result(n, dim, device=True)
    s.solve_batch(db, out=out)
    ts = []
    for _ in range(9):
        s.solve_batch(db, out=out); ts.append(out.kernel_time)
    ts.sort()
    print(f"{os.path.basename(os.environ['TB_LIB_PATH']):14s} {fam:8s} x{n:6d}: median {ts[4]*1e3:8.3f} ms  best {ts[0]*1e3:8.3f} ms", flush=True)
"""
for r in range(rounds):
    for lib in libs:
        env = dict(os.environ, TB_LIB_PATH=os.path.abspath(lib), AB_WORK=work)
        p = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
        print(p.stdout.strip() or p.stderr[-600:], flush=True)
