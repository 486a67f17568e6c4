"""Launch order (tb_context_set_order / LaunchOrder, tron_order.cu): ranking
a batch by the start projected-gradient norm changes which problems start
first, never what is computed -- every SolveReport field and the flop
counters are bitwise the oracle's in every order, form and path."""
import os

import numpy as np
import pytest

from conftest import assert_bitwise, host
from oracle import pyoracle as po
from paper_2106_14995_b200 import KernelForm, LaunchOrder, ProblemBatch, Solver, synth

pytestmark = pytest.mark.gpu
W = os.cpu_count() or 8


def _dev(b):
    import torch

    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    return ProblemBatch(b.family, b.dim, t(b.lower), t(b.upper), t(b.params) if b.params is not None else None,
                        t(b.x0))


CASES = [("branch", 6, 65536, KernelForm.AUTO), ("branch", 4, 20467, KernelForm.AUTO),
         ("branch", 4, 9000, KernelForm.WARP), ("ncvx", 4, 32768, KernelForm.AUTO), ("ncvx", 8, 12000, KernelForm.AUTO),
         ("ncvx", 16, 6000, KernelForm.AUTO), ("ncvx", 40, 600, KernelForm.AUTO), ("ncvx", 100, 96, KernelForm.AUTO),
         ("hs45", 12, 64, KernelForm.AUTO), ("boxqp", 8, 5000, KernelForm.AUTO)]


@pytest.mark.parametrize("fam,d,N,form", CASES)
def test_orders_bitwise_device_resident(fam, d, N, form):
    b = synth.make(fam, N, d, seed=11 + d)
    ref = po.solve_batch(b, impl="oracle", workers=W)
    db = _dev(b)
    for order in (LaunchOrder.START_PG, LaunchOrder.INDEX, LaunchOrder.AUTO, LaunchOrder.CALLER):
        s = Solver((0,), form=form, order=order)
        try:
            out = Solver.alloc_result(N, d, device=True)
            s.solve_batch(db, out=out)
            assert_bitwise(out, ref, label=f"{fam}{d} x{N} {form.name} {order.name}")
        finally:
            s.close()


@pytest.mark.parametrize("fam,d,N", [("branch", 6, 20000), ("ncvx", 8, 9000), ("ncvx", 48, 300)])
def test_start_pg_order_host_buffers_and_flops(fam, d, N):
    b = synth.make(fam, N, d, seed=3)
    ref = po.solve_batch(b, impl="oracle", workers=W)
    s = Solver((0,), order=LaunchOrder.START_PG)
    try:
        assert_bitwise(s.solve_batch(b), ref, label=f"{fam}{d} host")
        r = s.solve_batch(b, count_flops=True)
        assert_bitwise(r, ref, label=f"{fam}{d} counted")
        assert np.array_equal(host(r.flops), ref.flops)
        assert_bitwise(s.solve_batch(_dev(b)), ref, label=f"{fam}{d} device")
    finally:
        s.close()


def test_start_pg_order_two_partitions_and_async_streams():
    import torch

    b = synth.branch(30000, 6, seed=4)
    ref = po.solve_batch(b, impl="oracle", workers=W)
    s = Solver((0, 0), order=LaunchOrder.START_PG)
    try:
        assert_bitwise(s.solve_batch(b), ref, label="G=2 ranked")
    finally:
        s.close()
    s = Solver((0,), order=LaunchOrder.START_PG)
    try:
        db = _dev(b)
        dev = torch.device("cuda", 0)
        ss = [torch.cuda.Stream(dev) for _ in range(3)]
        outs = [Solver.alloc_result(b.count, 6, device=True) for _ in ss]
        for st, o in zip(ss, outs):
            s.solve_batch(db, out=o, stream=st.cuda_stream)
        torch.cuda.synchronize()
        for k, o in enumerate(outs):
            assert_bitwise(o, ref, label=f"ranked async {k}")
    finally:
        s.close()


def test_caller_order_host_buffers():
    """TB_ORDER_CALLER: the caller's own order as one launch (host buffers go
    over whole, like a ranked batch)."""
    b = synth.branch(20000, 6, seed=9)
    s = Solver((0,), order=LaunchOrder.CALLER)
    try:
        assert_bitwise(s.solve_batch(b), po.solve_batch(b, impl="oracle", workers=W), label="caller order")
    finally:
        s.close()


@pytest.mark.parametrize("n", [1, 2, 3, 31, 33, 257])
def test_start_pg_order_small_and_odd_sizes(n):
    b = synth.branch(n, 6, seed=n)
    ref = po.solve_batch(b, impl="oracle", workers=W)
    s = Solver((0,), order=LaunchOrder.START_PG)
    try:
        assert_bitwise(s.solve_batch(b), ref, label=f"ranked host n={n}")
        assert_bitwise(s.solve_batch(_dev(b)), ref, label=f"ranked device n={n}")
    finally:
        s.close()


def test_ranked_batch_reports_the_first_failure_in_input_order():
    """batch.hpp:75-76 in a ranked launch: the error names the first failing
    problem in INPUT order, whatever order the problems were solved in."""
    b = synth.branch(30000, 6, seed=12)
    lo = np.array(b.lower, copy=True)
    for i in (29000, 17, 5000):
        lo[i, 1] = b.upper[i, 1] + 0.5
    b = ProblemBatch(b.family, 6, lo, b.upper, b.params, b.x0)
    ref = po.solve_batch(b, impl="oracle", workers=W)
    for order in (LaunchOrder.START_PG, LaunchOrder.AUTO):
        s = Solver((0,), order=order)
        try:
            with pytest.raises(Exception, match="problem 17"):
                s.solve_batch(b)
            out = Solver.alloc_result(b.count, 6, device=True)
            with pytest.raises(Exception, match="problem 17"):
                s.solve_batch(_dev(b), out=out)
            assert np.array_equal(host(out.status), ref.status)
        finally:
            s.close()


def test_set_order_rejects_unknown():
    s = Solver((0,))
    try:
        with pytest.raises(ValueError, match="unknown launch order"):
            s.set_order(7)
    finally:
        s.close()
