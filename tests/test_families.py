"""Problem families (host twins = the device's shared code): derivative
oracles (SPEC acceptance 4), twins of the reference's own problems bitwise,
and the branch flows against an independent complex pi-model oracle."""
import ctypes as C

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2106_14995_b200 import Family, synth

needs_ref = pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref not built")


def fd_grad(f, x, h=1e-6):
    g = np.zeros_like(x)
    for i in range(len(x)):
        xp, xm = x.copy(), x.copy()
        xp[i] += h
        xm[i] -= h
        g[i] = (f(xp) - f(xm)) / (2 * h)
    return g


def rel_err(a, b):
    return np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b)))


@pytest.mark.parametrize("fam,d", [("ncvx", 3), ("ncvx", 8), ("branch", 4), ("branch", 6), ("boxqp", 5), ("hs45", 6)])
def test_derivatives_match_finite_differences(fam, d):
    """gradient vs central differences of f (<= 1e-6 rel), Hessian vs central
    differences of the gradient (<= 1e-5 rel), at 50 random interior points."""
    b = synth.make(fam, 50, d)
    rng = np.random.default_rng(1)
    for k in range(50):
        lo, up = b.lower[k], b.upper[k]
        lo_f = np.where(np.isfinite(lo), lo, -2.0)
        up_f = np.where(np.isfinite(up), up, 2.0)
        x = lo_f + (up_f - lo_f) * rng.uniform(0.2, 0.8, size=d)
        prm = None if b.params is None else b.params[k]
        f0, g0, H0 = po.family_eval(int(b.family), d, x, prm)
        f = lambda z: po.family_eval(int(b.family), d, z, prm)[0]  # noqa: E731
        g = lambda z: po.family_eval(int(b.family), d, z, prm)[1]  # noqa: E731
        assert rel_err(g0, fd_grad(f, x)) <= 1e-6
        Hfd = np.stack([fd_grad(lambda z: g(z)[i], x) for i in range(d)])
        assert rel_err(H0, Hfd) <= 1e-5
        assert np.array_equal(H0, H0.T)  # symmetric bit-for-bit


@needs_ref
@pytest.mark.parametrize("d", [1, 2, 3, 8, 17, 32])
def test_hs45_twin_bitwise_equals_reference(d):
    """tb_families.h hs45 == Hs45Problem::eval_* (batch.hpp:133-164)."""
    rng = np.random.default_rng(d)
    x = rng.uniform(0.1, 2.0, size=d)
    f, g, H = po.family_eval(Family.HS45, d, x)
    rf, rg, rH = C.c_double(), np.zeros(d), np.zeros(d * d)
    po.ref_lib().fn("hs45_eval")(d, x.ctypes.data_as(po.dp), C.byref(rf), rg.ctypes.data_as(po.dp),
                                 rH.ctypes.data_as(po.dp))
    assert f == rf.value and np.array_equal(g, rg) and np.array_equal(H, rH.reshape(d, d).T)


@needs_ref
def test_boxqp_twin_bitwise_equals_reference():
    """tb_families.h boxqp == make_quadratic (boxqp_oracle.hpp:44-62)."""
    b = synth.boxqp(20, 6)
    for k in range(20):
        x = b.x0[k].copy()
        x[2] = b.params[k, 36 + 2]  # one exact zero in d = x - c exercises the gemv zero-skip
        f, g, _ = po.family_eval(Family.BOXQP, 6, x, b.params[k])
        rf, rg = C.c_double(), np.zeros(6)
        Hq = np.ascontiguousarray(b.params[k, :36])
        c = np.ascontiguousarray(b.params[k, 36:])
        po.ref_lib().fn("boxqp_eval")(6, Hq.ctypes.data_as(po.dp), c.ctypes.data_as(po.dp), x.ctypes.data_as(po.dp),
                                      C.byref(rf), rg.ctypes.data_as(po.dp))
        assert f == rf.value and np.array_equal(g, rg)


def test_branch_flows_match_complex_pi_model():
    """Eq. (2i)-(2l) flows == V_i conj(I_ij) of the pi model
    computed with complex arithmetic (independent oracle), within 1e-10."""
    rng = np.random.default_rng(3)
    n = 200
    r, x, bc = rng.uniform(0.001, 0.05, n), rng.uniform(0.01, 0.3, n), rng.uniform(0, 0.1, n)
    tap, shift = rng.uniform(0.95, 1.05, n), rng.uniform(-0.1, 0.1, n)
    coef = synth.pi_model(r, x, bc, tap, shift)
    vi, vj = rng.uniform(0.9, 1.1, n), rng.uniform(0.9, 1.1, n)
    ti, tj = rng.uniform(-0.5, 0.5, n), rng.uniform(-0.5, 0.5, n)
    F = synth.branch_flows(coef, vi, vj, ti, tj)
    y = 1.0 / (r + 1j * x)
    tau = tap * np.exp(1j * shift)
    Yff, Yft, Ytf, Ytt = (y + 1j * bc / 2) / tap**2, -y / np.conj(tau), -y / tau, y + 1j * bc / 2
    Vi, Vj = vi * np.exp(1j * ti), vj * np.exp(1j * tj)
    Sij = Vi * np.conj(Yff * Vi + Yft * Vj)
    Sji = Vj * np.conj(Ytf * Vi + Ytt * Vj)
    ref = np.stack([Sij.real, Sij.imag, Sji.real, Sji.imag], axis=-1)
    assert np.max(np.abs(F - ref)) <= 1e-10
    # lossless line (r = 0, no shunt, tap 1): p_ij + p_ji = 0
    c0 = synth.pi_model(np.zeros(1), np.ones(1), np.zeros(1), np.ones(1))
    F0 = synth.branch_flows(c0, np.array([1.02]), np.array([0.97]), np.array([0.1]), np.array([-0.2]))
    assert abs(F0[0, 0] + F0[0, 2]) < 1e-14


def test_branch_device_family_flows_equal_numpy():
    """The family's own flows (portable sincos) agree with numpy's at 1e-12:
    f == 0 and grad == 0 when tilde = flows and lambda = 0."""
    b = synth.branch(5, 4, seed=11)
    for k in range(5):
        x = np.array([1.01, 0.98, 0.05, -0.03])
        P = b.params[k].copy()
        P[8:12] = 0.0
        P[20:22] = 0.0
        P[26:28] = 0.0
        P[16:20] = synth.branch_flows(P[:8], x[0], x[1], x[2], x[3])
        P[24:26] = x[:2] ** 2
        P[30:32] = x[2:4]
        f, g, _ = po.family_eval(Family.BRANCH, 4, x, P)
        assert abs(f) < 1e-20 and np.max(np.abs(g)) < 1e-10
