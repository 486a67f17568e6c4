"""Generate the committed golden fixtures from the REFERENCE ITSELF.

Runs the unmodified reference headers (compiled into oracle/_ref/libtronref.so
by `make -C oracle ref`; needs /root/reference) on seeded synthetic batches and
stores inputs + every SolveReport field in tests/golden/*.npz.  The GPU box has
no /root/reference, so these fixtures carry the reference's answers there.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import pyoracle  # noqa: E402
from paper_2106_14995_b200 import synth  # noqa: E402

CASES = {
    # BASELINE configs[0] (C1): 1,024 random nonconvex d=4 problems, seed 1
    "c1_ncvx_d4": lambda: synth.ncvx(1024, 4, seed=1),
    # C2 shape (d=6 branch AL subproblems), first 2,048 problems of seed 2
    "c2_branch6": lambda: synth.branch(2048, 6, seed=2),
    "branch4": lambda: synth.branch(1024, 4, seed=7),
    # C3 sweep shapes at fixture size
    "c3_ncvx_d8": lambda: synth.ncvx(256, 8, seed=11),
    "c3_ncvx_d16": lambda: synth.ncvx(64, 16, seed=19),
    "c3_ncvx_d32": lambda: synth.ncvx(32, 32, seed=35),
    # d > 32: the block kernel (D = 64 / 128 threads)
    "c3_ncvx_d64": lambda: synth.ncvx(16, 64, seed=67),
    "c3_ncvx_d128": lambda: synth.ncvx(8, 128, seed=131),
    "boxqp_d48": lambda: synth.boxqp(16, 48, seed=53),
    # tests/unit/tron_test.cpp:196-212 shapes
    "boxqp_d4": lambda: synth.boxqp(256, 4, seed=5),
    "hs45_d8": lambda: synth.hs45(4, 8),
    "hs45_d64": lambda: synth.hs45(2, 64),  # batch.hpp:15 kDefaultCapacity
}


def main():
    assert pyoracle.ref_available(), "build oracle/_ref first: make -C oracle ref"
    only = set(sys.argv[1:])  # optional: regenerate just these fixtures
    for name, mk in CASES.items():
        if only and name not in only:
            continue
        b = mk()
        r = pyoracle.solve_batch(b, impl="ref", workers=os.cpu_count() or 1)
        assert r.rc == 0, (name, pyoracle.last_error())
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"), family=int(b.family), dim=int(b.dim), x0=b.x0, lower=b.lower,
            upper=b.upper, params=(b.params if b.params is not None else np.zeros((b.count, 0))),
            x_star=r.x_star, f_star=r.f_star, pg_norm=r.pg_norm, status=r.status, iterations=r.iterations,
            cg_iterations=r.cg_iterations, f_evals=r.f_evals)
        print(f"{name}: {b.count} problems, status counts {np.bincount(r.status).tolist()}")


if __name__ == "__main__":
    main()
