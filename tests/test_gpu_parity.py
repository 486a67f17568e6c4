"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Exact mode is bit-identical for every SolveReport field."""
import numpy as np
import pytest

from conftest import assert_bitwise, host
from oracle import pyoracle as po
from paper_2106_14995_b200 import SolveStatus, TronConfig, synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 6, 7, 8, 12, 16, 24, 32])
def test_ncvx_bitwise(solver, d):
    n = 1024 if d <= 8 else 128
    b = synth.ncvx(n, d, seed=3 + d)
    res = solver.solve_batch(b)
    ref = po.solve_batch(b, impl="oracle", workers=8)
    assert_bitwise(res, ref, label=f"ncvx d={d}")
    assert np.array_equal(host(res.flops), ref.flops)


def test_c1_ncvx_d4_1024(solver):
    """BASELINE configs[0]: 1,024 random nonconvex d=4 problems."""
    b = synth.ncvx(1024, 4, seed=1)
    res = solver.solve_batch(b)
    ref = po.solve_batch(b, impl="oracle")
    assert_bitwise(res, ref, label="C1")
    assert (host(res.status) == 0).all()


@pytest.mark.parametrize("dim", [4, 6])
def test_branch_bitwise(solver, dim):
    b = synth.branch(8192, dim, seed=2)
    res = solver.solve_batch(b)
    ref = po.solve_batch(b, impl="oracle", workers=8)
    assert_bitwise(res, ref, label=f"branch{dim}")
    assert np.array_equal(host(res.flops), ref.flops)


@pytest.mark.parametrize("d", [1, 2, 4, 8, 16, 32])
def test_hs45(solver, d):
    """SPEC acceptance 1: x*_i = i, f* = 120 - n!"""
    b = synth.hs45(4, d)
    res = solver.solve_batch(b)
    ref = po.solve_batch(b, impl="oracle")
    assert_bitwise(res, ref, label=f"hs45 {d}")
    xs = host(res.x_star)
    assert (host(res.status) == 0).all()
    assert np.abs(xs - np.arange(1, d + 1)).max() <= 1e-6
