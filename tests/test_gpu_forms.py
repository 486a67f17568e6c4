"""Kernel forms (tb_context_set_form / KernelForm) against the CPU oracle, bit
for bit, and the context's ordering of overlapping async solves.

Every form runs the reference's solve (tron.hpp:453-549) with the same
operation sequence, so every SolveReport field and the flop counters must
agree with the oracle whichever form solves a batch."""
import os

import numpy as np
import pytest

from conftest import assert_bitwise, forced_form, host
from oracle import pyoracle as po
from paper_2106_14995_b200 import KernelForm, ProblemBatch, Solver, TronConfig, synth

pytestmark = pytest.mark.gpu
W = os.cpu_count() or 8


def _dev(b):
    import torch

    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    return ProblemBatch(b.family, b.dim, t(b.lower), t(b.upper), t(b.params) if b.params is not None else None,
                        t(b.x0))


@pytest.mark.parametrize("fam,d", [("ncvx", 1), ("ncvx", 3), ("ncvx", 5), ("ncvx", 8), ("branch", 4), ("branch", 6),
                                   ("boxqp", 2), ("boxqp", 8), ("hs45", 4), ("hs45", 8)])
def test_warp_form_forced_bitwise_with_flops(solver, fam, d):
    b = synth.make(fam, 2000 if fam != "hs45" else 8, d, seed=40 + d)
    ref = po.solve_batch(b, impl="oracle", workers=W)
    with forced_form(solver, KernelForm.WARP):
        res = solver.solve_batch(b, count_flops=True)
        assert_bitwise(res, ref, label=f"warp {fam}{d}")
        assert np.array_equal(host(res.flops), ref.flops), f"warp {fam}{d} flops"
        assert_bitwise(solver.solve_batch(b), ref, label=f"warp {fam}{d} (no count)")


@pytest.mark.parametrize("cfg", [TronConfig(max_iter=3), TronConfig(tol_pg=1e-9)])
def test_thread_form_forced_small_batches(solver, cfg):
    with forced_form(solver, KernelForm.THREAD):
        for b in (synth.ncvx(777, 4, seed=4), synth.branch(777, 4, seed=4)):
            assert_bitwise(solver.solve_batch(b, cfg=cfg), po.solve_batch(b, cfg=cfg, impl="oracle", workers=W),
                           label=f"thread {cfg}")


def test_overlapping_async_block_kernel_solves(solver):
    """async block-kernel solves on different streams share the
    context workspace (work counter, Hessian slices); the context orders them
    on an event, so all are exact."""
    import torch

    b = synth.ncvx(200, 40, seed=3)
    ref = po.solve_batch(b, impl="oracle", workers=W)
    db = _dev(b)
    dev = torch.device("cuda", 0)
    ss = [torch.cuda.Stream(dev) for _ in range(3)]
    outs = [Solver.alloc_result(b.count, 40, device=True) for _ in ss]
    for s, o in zip(ss, outs):
        solver.solve_batch(db, out=o, stream=s.cuda_stream)
    torch.cuda.synchronize()
    for k, o in enumerate(outs):
        assert_bitwise(o, ref, label=f"async block {k}")


def test_overlapping_async_warp_and_thread_solves(solver):
    import torch

    dev = torch.device("cuda", 0)
    for b in (synth.branch(20000, 6, seed=8), synth.branch(20000, 4, seed=8)):
        ref = po.solve_batch(b, impl="oracle", workers=W)
        db = _dev(b)
        ss = [torch.cuda.Stream(dev) for _ in range(2)]
        outs = [Solver.alloc_result(b.count, b.dim, device=True) for _ in ss]
        for s, o in zip(ss, outs):
            solver.solve_batch(db, out=o, stream=s.cuda_stream)
        torch.cuda.synchronize()
        for k, o in enumerate(outs):
            assert_bitwise(o, ref, label=f"async d={b.dim} {k}")


def test_block_form_forced_at_small_d_and_warp_at_d24(solver):
    b = synth.ncvx(200, 12, seed=5)
    ref = po.solve_batch(b, impl="oracle", workers=W)
    with forced_form(solver, KernelForm.BLOCK):
        assert_bitwise(solver.solve_batch(b), ref, label="block d=12")
    b24 = synth.ncvx(100, 24, seed=6)
    with forced_form(solver, KernelForm.WARP):
        assert_bitwise(solver.solve_batch(b24), po.solve_batch(b24, impl="oracle", workers=W), label="warp d=24")


def test_set_form_rejects_unknown():
    s = Solver((0,))
    try:
        with pytest.raises(ValueError, match="unknown kernel form"):
            s.set_form(2)
    finally:
        s.close()


def test_fast_forward_modes_identical_reports():
    """fast_forward 0 / 1 / 2 (replay / skip + credit the reference's flops /
    skip + count executed flops): every SolveReport field identical; the
    credited count equals the replayed count, the executed count is smaller
    exactly when something was skipped."""
    b = synth.branch(8192, 6, seed=5)
    rs = []
    for ff in (0, 1, 2):
        s = Solver((0,), fast_forward=ff)
        try:
            rs.append(s.solve_batch(b, count_flops=True))
        finally:
            s.close()
    assert_bitwise(rs[1], rs[0], label="ff1 vs ff0")
    assert_bitwise(rs[2], rs[0], label="ff2 vs ff0")
    f0, f1, f2 = (host(r.flops) for r in rs)
    assert np.array_equal(f0, f1)
    assert (f2 <= f1).all() and (f2 < f1).any()
