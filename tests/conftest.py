import contextlib
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


FIELDS = ("x_star", "f_star", "pg_norm", "status", "iterations", "cg_iterations", "f_evals")


def host(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)


def assert_bitwise(res, ref, fields=FIELDS, label=""):
    """Exact (bitwise) equality of every SolveReport field; NaNs compare equal."""
    for k in fields:
        a, b = host(getattr(res, k)), np.asarray(getattr(ref, k))
        assert a.shape == b.shape, (label, k, a.shape, b.shape)
        if a.dtype.kind == "f":
            eq = (a.view(np.int64) == b.view(np.int64)) | (np.isnan(a) & np.isnan(b))
        else:
            eq = a == b
        if not eq.all():
            eqp = eq.reshape(eq.shape[0], -1).all(axis=1)
            i = int(np.argmin(eqp))
            raise AssertionError(f"{label}: field {k} differs at problem {i}: {a[i]!r} vs {b[i]!r} "
                                 f"({int((~eqp).sum())} problems differ)")


@contextlib.contextmanager
def forced_form(solver, form):
    """Run the block with the session solver forced to a kernel form."""
    from paper_2106_14995_b200 import KernelForm

    solver.set_form(form)
    try:
        yield solver
    finally:
        solver.set_form(KernelForm.AUTO)


@pytest.fixture(scope="session")
def solver():
    from paper_2106_14995_b200 import Solver

    s = Solver((0,))
    yield s
    s.close()
