"""tb_solve_batch_packed: the per-chunk pack / unpack callbacks the C++
drop-in uses (include/tronbatch_gpu/solve_batch.hpp) instead of packing the
whole batch up front.  Through ctypes here: every SolveReport field bitwise
equal to the CPU oracle, callbacks in problem order over the whole batch, and
the reference's error behaviour (batch.hpp:75-76: the first problem that
would have thrown turns the call into TB_E_PROBLEM)."""
import ctypes as C
import os

import numpy as np
import pytest

from conftest import assert_bitwise
from oracle import pyoracle as po
from paper_2106_14995_b200 import Solver, TronConfig, _lib as L, synth

pytestmark = pytest.mark.gpu
W = os.cpu_count() or 8


class _Out:
    pass


def _packed(solver, b, cfg=None):
    lib = L.load()
    N, n = b.count, b.dim
    np_ = int(lib.tb_family_nparams(int(b.family), n))
    x0, lo, up = (np.ascontiguousarray(a, dtype=np.float64) for a in (b.x0, b.lower, b.upper))
    prm = None if b.params is None else np.ascontiguousarray(b.params, dtype=np.float64)
    out = _Out()
    out.x_star = np.full((N, n), np.nan)
    out.f_star, out.pg_norm, out.wall = np.full(N, np.nan), np.full(N, np.nan), np.zeros(N)
    out.status, out.iterations = np.full(N, -1, np.int32), np.full(N, -1, np.int32)
    out.cg_iterations, out.f_evals = np.full(N, -1, np.int64), np.full(N, -1, np.int64)
    calls = []

    def view(p, shape, dt):
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(np.ctypeslib.as_ctypes_type(dt))), shape=shape)

    def pack(_u, a, e, px0, plo, pup, pprm):
        calls.append(("pack", a, e))
        m = e - a
        view(px0, (m, n), np.float64)[:] = x0[a:e]
        view(plo, (m, n), np.float64)[:] = lo[a:e]
        view(pup, (m, n), np.float64)[:] = up[a:e]
        if np_ > 0:
            view(pprm, (m, np_), np.float64)[:] = prm[a:e, :np_]
        else:
            assert not pprm

    def unpack(_u, a, e, rp):
        calls.append(("unpack", a, e))
        r, m = rp.contents, e - a
        assert not r.flops
        out.x_star[a:e] = view(r.x_star, (m, n), np.float64)
        out.f_star[a:e] = view(r.f_star, (m,), np.float64)
        out.pg_norm[a:e] = view(r.pg_norm, (m,), np.float64)
        out.status[a:e] = view(r.status, (m,), np.int32)
        out.iterations[a:e] = view(r.iterations, (m,), np.int32)
        out.cg_iterations[a:e] = view(r.cg_iterations, (m,), np.int64)
        out.f_evals[a:e] = view(r.f_evals, (m,), np.int64)
        out.wall[a:e] = view(r.wall_time, (m,), np.float64)

    pk, upk = L.PACK_FN(pack), L.UNPACK_FN(unpack)
    agg = L.BatchResultC()
    c = (cfg or TronConfig()).to_c()
    rc = lib.tb_solve_batch_packed(solver._ctx, int(b.family), n, N, C.byref(c), pk, upk, None, C.byref(agg))
    return rc, out, calls, agg


def _covers(calls, kind, N):
    rs = [(a, e) for k, a, e in calls if k == kind]
    assert rs[0][0] == 0 and rs[-1][1] == N, rs
    assert all(rs[i][1] == rs[i + 1][0] for i in range(len(rs) - 1)), rs  # problem order, no gaps
    return len(rs)


@pytest.mark.parametrize("fam,d,N", [("branch", 6, 65536), ("branch", 4, 20467), ("ncvx", 8, 9000),
                                     ("hs45", 5, 64), ("ncvx", 40, 300)])
def test_packed_bitwise_vs_oracle(solver, fam, d, N):
    b = synth.make(fam, N, d, seed=7 + d)
    rc, out, calls, agg = _packed(solver, b)
    assert rc == L.TB_OK, L.last_error()
    assert_bitwise(out, po.solve_batch(b, impl="oracle", workers=W), label=f"packed {fam}{d}")
    nch = _covers(calls, "pack", N)
    assert _covers(calls, "unpack", N) == nch
    if N >= 65536:
        assert nch > 1  # pipelined in chunks
    assert agg.n_partitions == 1 and agg.batch_wall_time > 0.0 and (out.wall > 0).all()


def test_packed_two_partitions_on_one_gpu():
    b = synth.branch(30000, 6, seed=3)
    s = Solver((0, 0))
    try:
        rc, out, calls, agg = _packed(s, b)
    finally:
        s.close()
    assert rc == L.TB_OK
    assert_bitwise(out, po.solve_batch(b, impl="oracle", workers=W), label="packed G=2")
    _covers(calls, "pack", b.count)
    assert agg.n_partitions == 2


def test_packed_first_failure_is_the_error(solver):
    b = synth.ncvx(12000, 6, seed=5)
    lo = np.array(b.lower, copy=True)
    for i in (7001, 9000):  # invalid bounds: the reference throws invalid_argument at the first
        lo[i, 2] = b.upper[i, 2] + 1.0
    b = type(b)(b.family, b.dim, lo, b.upper, b.params, b.x0)
    rc, out, _, _ = _packed(solver, b)
    assert rc == L.TB_E_PROBLEM
    assert "problem 7001" in L.last_error()
    ok = np.ones(b.count, bool)
    ok[[7001, 9000]] = False
    ref = po.solve_batch(b, impl="oracle", workers=W)
    assert np.array_equal(out.status, ref.status)
    assert np.array_equal(out.x_star[ok].view(np.int64), ref.x_star[ok].view(np.int64))


def test_packed_rejects_null_callbacks(solver):
    lib = L.load()
    c = TronConfig().to_c()
    agg = L.BatchResultC()
    rc = lib.tb_solve_batch_packed(solver._ctx, 3, 4, 10, C.byref(c), L.PACK_FN(), L.UNPACK_FN(), None,
                                   C.byref(agg))
    assert rc == L.TB_E_INVALID_ARGUMENT
