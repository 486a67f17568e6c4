"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Exact mode is bit-identical for every SolveReport field."""
import numpy as np
import pytest

from conftest import assert_bitwise, forced_form, host
from oracle import pyoracle as po
from paper_2106_14995_b200 import KernelForm, SolveStatus, TronConfig, synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 6, 7, 8, 12, 16, 24, 32])
def test_ncvx_bitwise(solver, d):
    n = 1024 if d <= 8 else 128
    b = synth.ncvx(n, d, seed=3 + d)
    res = solver.solve_batch(b, count_flops=True)
    ref = po.solve_batch(b, impl="oracle", workers=8)
    assert_bitwise(res, ref, label=f"ncvx d={d}")
    assert np.array_equal(host(res.flops), ref.flops)
    plain = solver.solve_batch(b)  # non-counting kernel variant: same results
    assert_bitwise(plain, ref, label=f"ncvx d={d} (no count)")


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
    res = solver.solve_batch(b, count_flops=True)
    ref = po.solve_batch(b, impl="oracle", workers=8)
    assert_bitwise(res, ref, label=f"branch{dim}")
    assert np.array_equal(host(res.flops), ref.flops)


@pytest.mark.parametrize("d", [1, 2, 4, 8, 16, 32])
def test_hs45(solver, d):  # d > 32: test_block_kernel_boxqp_hs45_bitwise
    """SPEC acceptance 1: x*_i = i, f* = 120 - n!"""
    b = synth.hs45(4, d)
    res = solver.solve_batch(b)
    ref = po.solve_batch(b, impl="oracle")
    assert_bitwise(res, ref, label=f"hs45 {d}")
    xs = host(res.x_star)
    assert (host(res.status) == 0).all()
    assert np.abs(xs - np.arange(1, d + 1)).max() <= 1e-6


# ---------------------------------------------------------------- fixtures
import glob  # noqa: E402
import os  # noqa: E402
from types import SimpleNamespace  # noqa: E402

from conftest import FIELDS  # noqa: E402
from paper_2106_14995_b200 import (  # noqa: E402
    EvaluationError, ProblemBatch, Solver, SolveStatus, TronConfig)

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "*.npz")))


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_device_matches_reference_golden(solver, path):
    """Fixtures hold the REFERENCE's own outputs (tests/golden/make_golden.py)."""
    g = np.load(path)
    prm = g["params"] if g["params"].shape[1] else None
    b = ProblemBatch(int(g["family"]), int(g["dim"]), g["lower"], g["upper"], prm, g["x0"])
    res = solver.solve_batch(b)
    assert_bitwise(res, SimpleNamespace(**{k: g[k] for k in FIELDS}), label=os.path.basename(path))


def test_c2_full_size_bitwise(solver):
    """BASELINE configs[1] at full size: 65,536 branch6 problems, every field
    bit-identical to the CPU oracle (restatement pinned to the reference)."""
    b = synth.branch(65536, 6, seed=2)
    res = solver.solve_batch(b)
    ref = po.solve_batch(b, impl="oracle", workers=os.cpu_count() or 8)
    assert_bitwise(res, ref, label="C2 65536")
    st = host(res.status)
    assert (st <= 1).all() and (st == 1).mean() < 0.02


def test_boxqp_matches_bruteforce_active_set_oracle(solver):
    """SPEC acceptance 5 / tron_test.cpp:196-212 at 50 problems."""
    import ctypes as C

    b = synth.boxqp(50, 4, seed=21)
    res = solver.solve_batch(b)
    assert (host(res.status) == 0).all()
    xs = host(res.x_star)
    for k in range(50):
        H = np.ascontiguousarray(b.params[k, :16])
        c = np.ascontiguousarray(b.params[k, 16:])
        lo, up = np.ascontiguousarray(b.lower[k]), np.ascontiguousarray(b.upper[k])
        x = np.zeros(4)
        if po.ref_available():
            f = po.ref_lib().fn("boxqp_oracle")
            assert f(4, H.ctypes.data_as(po.dp), c.ctypes.data_as(po.dp), lo.ctypes.data_as(po.dp),
                     up.ctypes.data_as(po.dp), x.ctypes.data_as(po.dp)) == 0
            assert np.max(np.abs(xs[k] - x)) <= 1e-6


def test_empty_batch(solver):
    b = synth.ncvx(0, 4)
    res = solver.solve_batch(b)
    assert host(res.status).shape == (0,)


def test_start_outside_box_and_infinite_bounds(solver):
    """tron.hpp:473 (x0 is projected, never rejected); tron.hpp:17 (+-inf)."""
    b = synth.boxqp(256, 5, seed=8)
    b.lower[::3, 1] = -np.inf
    b.upper[::4, 2] = np.inf
    x0 = b.x0 * 5.0
    res = solver.solve_batch(b, x0)
    ref = po.solve_batch(b, x0, impl="oracle")
    assert_bitwise(res, ref, label="outside/inf")
    xs = host(res.x_star)
    assert (xs >= b.lower).all() and (xs <= b.upper).all()


@pytest.mark.parametrize("cfg", [TronConfig(max_iter=1), TronConfig(delta0=0.3), TronConfig(tol_pg=1e-9),
                                 TronConfig(cg_tol=0.5, mu0=0.1, interp_factor=0.25),
                                 TronConfig(sigma1=0.1, sigma2=0.3, sigma3=2.0, eta0=0.01, delta_max=5.0)])
def test_config_variants_bitwise(solver, cfg):
    for b in (synth.ncvx(256, 6, seed=4), synth.branch(256, 6, seed=4), synth.hs45(2, 8)):
        assert_bitwise(solver.solve_batch(b, cfg=cfg), po.solve_batch(b, cfg=cfg, impl="oracle"), label=str(cfg))


def test_iteration_limit_status(solver):
    """tron_test.cpp:242-249 intent (IterLimit at max_iter=1) on a problem that
    does not converge in one iteration."""
    b = synth.ncvx(64, 8, seed=2)
    res = solver.solve_batch(b, cfg=TronConfig(max_iter=1))
    st, it = host(res.status), host(res.iterations)
    assert ((st == 1) & (it == 1)).sum() > 0
    assert_bitwise(res, po.solve_batch(b, cfg=TronConfig(max_iter=1), impl="oracle"))


def test_nan_hessian_factorization_failed(solver):
    """tron_test.cpp:251-266: H = [[1, 0], [0, NaN]] with a zero second
    gradient component (the gemv zero-skip, dense.hpp:110, keeps the Cauchy
    model finite); the NaN pivot fails every shift until the cap
    (dense.hpp:197-199) -> FactorizationFailed."""
    H = np.array([1.0, 0.0, 0.0, np.nan])  # column-major
    c = np.array([0.0, 0.5])
    prm = np.tile(np.concatenate([H, c]), (3, 1))
    b = ProblemBatch(1, 2, np.full((3, 2), -1.0), np.full((3, 2), 1.0), prm, np.tile([0.5, 0.5], (3, 1)))
    res = solver.solve_batch(b)
    ref = po.solve_batch(b, impl="oracle")
    assert_bitwise(res, ref, label="nan hessian")
    assert (host(res.status) == SolveStatus.FactorizationFailed).all()
    assert (host(res.iterations) == 1).all()


def test_evaluation_error_raises_like_reference(solver):
    """tron.hpp:190-194: a non-finite Cauchy model throws EvaluationError out
    of solve_batch (batch.hpp:75-76); the device raises the same type."""
    b = synth.boxqp(4, 3, seed=6)
    b.params[2, 0] = np.inf  # H(0,0) = inf in problem 2
    with pytest.raises(EvaluationError):
        solver.solve_batch(b)
    ref = po.solve_batch(b, impl="oracle")
    assert ref.rc == SolveStatus.EvaluationError


def test_invalid_bounds_raise(solver):
    b = synth.ncvx(4, 3)
    b.lower[1, 0] = b.upper[1, 0] + 1.0
    with pytest.raises(ValueError, match="lower bound exceeds upper bound"):
        solver.solve_batch(b)


def test_fast_forward_on_device_is_neutral():
    b = synth.branch(8192, 6, seed=5)
    a = Solver((0,), fast_forward=True).solve_batch(b, count_flops=True)
    z = Solver((0,), fast_forward=False).solve_batch(b, count_flops=True)
    assert_bitwise(a, z, label="device ff")
    assert np.array_equal(host(a.flops), host(z.flops))


def test_device_memspace_and_stream_async(solver):
    import torch

    b = synth.branch(4096, 6, seed=12)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    db = ProblemBatch(b.family, 6, t(b.lower), t(b.upper), t(b.params), t(b.x0))
    r1 = solver.solve_batch(db)  # blocking, device memspace
    s = torch.cuda.Stream(dev)
    out = Solver.alloc_result(b.count, 6, device=True)
    solver.solve_batch(db, out=out, stream=s.cuda_stream)
    s.synchronize()
    ref = po.solve_batch(b, impl="oracle", workers=8)
    assert_bitwise(r1, ref, label="device memspace")
    assert_bitwise(out, ref, label="async stream")


def test_dimension_over_device_capacity_rejected(solver):
    with pytest.raises(ValueError):
        solver.solve_batch(synth.ncvx(2, 129))


# ------------------------------------------------- d > 32: the block kernel
@pytest.mark.parametrize("d", [17, 24, 32, 33, 40, 64, 65, 100, 128])
def test_block_kernel_ncvx_bitwise(solver, d):
    """C3 sweep on the block kernel: D = 32 / 64 / 128 threads per problem, Hessian in
    the global workspace; every field, and the flop counters, bit-identical to the oracle."""
    asmem = "0"
    n = 48 if d <= 64 else 16
    b = synth.ncvx(n, d, seed=3 + d)
    res = solver.solve_batch(b, count_flops=True)
    ref = po.solve_batch(b, impl="oracle", workers=os.cpu_count() or 8)
    assert_bitwise(res, ref, label=f"ncvx d={d} asmem={asmem}")
    assert np.array_equal(host(res.flops), ref.flops)
    assert_bitwise(solver.solve_batch(b), ref, label=f"ncvx d={d} (no count)")


@pytest.mark.parametrize("d", [36, 64, 96])
def test_block_kernel_boxqp_hs45_bitwise(solver, d):
    for b in (synth.boxqp(24, d, seed=d), synth.hs45(2, min(d, 64))):
        assert_bitwise(solver.solve_batch(b), po.solve_batch(b, impl="oracle"), label=f"d={d} fam={b.family}")


def test_block_kernel_more_problems_than_resident_blocks(solver):
    """The persistent grid takes problems from a work counter: a batch several
    times the resident capacity, with config variants and outside starts."""
    b = synth.ncvx(2000, 40, seed=9)
    x0 = b.x0 * 3.0
    cfg = TronConfig(max_iter=7, cg_tol=0.3)
    res = solver.solve_batch(b, x0, cfg=cfg)
    assert_bitwise(res, po.solve_batch(b, x0, cfg=cfg, impl="oracle", workers=os.cpu_count() or 8), label="2000x40")


def test_block_kernel_device_memspace(solver):
    import torch

    b = synth.ncvx(64, 70, seed=70)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    db = ProblemBatch(b.family, 70, t(b.lower), t(b.upper), t(b.params), t(b.x0))
    assert_bitwise(solver.solve_batch(db), po.solve_batch(b, impl="oracle", workers=8), label="device d=70")


def test_hs45_acceptance_all_n(solver):
    """SPEC acceptance 1: n = 1..32 converge with x*_i = i and f* = 120 - n!."""
    import math

    for n in range(1, 33):
        res = solver.solve_batch(synth.hs45(1, n))
        assert host(res.status)[0] == 0
        assert np.abs(host(res.x_star)[0] - np.arange(1, n + 1)).max() <= 1e-6
        assert abs(host(res.f_star)[0] - (120.0 - math.factorial(n))) <= 1e-9 * max(1.0, math.factorial(n))


def test_cpp_dropin_against_reference_solve_batch():
    """include/tronbatch_gpu/solve_batch.hpp used exactly like the reference
    API (tests/cpp/gpu_dropin_test.cpp), compared with the reference's own
    CPU solve_batch in the same process (built with the reference headers)."""
    import subprocess

    exe = os.path.join(os.path.dirname(po.HERE), "oracle", "_ref", "gpu_dropin_test")
    if not os.path.exists(exe):
        pytest.skip("gpu_dropin_test not built (needs /root/reference at build time)")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stdout + p.stderr
    assert '"failed": 0' in p.stdout


# --------------------------------------- block kernel (d >= 21): edge cases
@pytest.mark.parametrize("cfg", [TronConfig(max_iter=1), TronConfig(delta0=0.3), TronConfig(tol_pg=1e-9),
                                 TronConfig(cg_tol=0.5, mu0=0.1, interp_factor=0.25),
                                 TronConfig(sigma1=0.1, sigma2=0.3, sigma3=2.0, eta0=0.01, delta_max=5.0)])
def test_block_kernel_config_variants_bitwise(solver, cfg):
    for b in (synth.ncvx(48, 24, seed=4), synth.ncvx(16, 70, seed=4), synth.hs45(2, 40)):
        assert_bitwise(solver.solve_batch(b, cfg=cfg), po.solve_batch(b, cfg=cfg, impl="oracle", workers=8),
                       label=f"d={b.dim} {cfg}")


def test_block_kernel_outside_box_and_infinite_bounds(solver):
    b = synth.boxqp(64, 40, seed=8)
    b.lower[::3, 1] = -np.inf
    b.upper[::4, 2] = np.inf
    x0 = b.x0 * 5.0
    res = solver.solve_batch(b, x0)
    assert_bitwise(res, po.solve_batch(b, x0, impl="oracle", workers=8), label="block outside/inf")


@pytest.mark.parametrize("d", [24, 40, 100])
def test_block_kernel_nan_hessian_factorization_failed(solver, d):
    """tron_test.cpp:251-266 at block-kernel sizes: a NaN diagonal entry with
    a zero gradient component -> FactorizationFailed at iteration 1."""
    H = np.eye(d).ravel(order="F")
    H[(d - 1) + (d - 1) * d] = np.nan
    c = np.zeros(d)
    c[-1] = 0.5
    prm = np.tile(np.concatenate([H, c]), (3, 1))
    b = ProblemBatch(1, d, np.full((3, d), -1.0), np.full((3, d), 1.0), prm, np.tile(np.full(d, 0.5), (3, 1)))
    b.x0[:, -1] = 0.5
    res = solver.solve_batch(b)
    assert_bitwise(res, po.solve_batch(b, impl="oracle"), label=f"nan hessian d={d}")
    assert (host(res.status) == SolveStatus.FactorizationFailed).all()


def test_block_kernel_evaluation_error_and_invalid_bounds(solver):
    b = synth.boxqp(4, 30, seed=6)
    b.params[2, 0] = np.inf
    with pytest.raises(EvaluationError):
        solver.solve_batch(b)
    b = synth.ncvx(4, 50)
    b.lower[1, 0] = b.upper[1, 0] + 1.0
    with pytest.raises(ValueError, match="lower bound exceeds upper bound"):
        solver.solve_batch(b)


@pytest.mark.parametrize("count", [0, 1, 3])
def test_block_kernel_tiny_batches(solver, count):
    b = synth.ncvx(count, 64, seed=12)
    res = solver.solve_batch(b)
    assert host(res.status).shape == (count,)
    if count:
        assert_bitwise(res, po.solve_batch(b, impl="oracle"), label=f"count={count}")


@pytest.mark.parametrize("d", [100, 128])
def test_block_kernel_large_free_systems_use_global_factor_slice(solver, d):
    """Wide bounds keep every variable free (nf = d > 108 at D = 128): the
    factor no longer fits the shared region and lives in the block's global
    fallback slice; results stay bit-identical."""
    # convex (one Newton step) and indefinite box QPs (several faces at nf = d)
    for b in (synth.boxqp(6, d, seed=d), synth.boxqp(6, d, seed=d + 1, spd_boost=-0.3)):
        b.lower[:] = -50.0
        b.upper[:] = 50.0
        res = solver.solve_batch(b, count_flops=True)
        ref = po.solve_batch(b, impl="oracle", workers=6)
        assert_bitwise(res, ref, label=f"wide bounds d={d} fam={b.family}")
        assert np.array_equal(host(res.flops), ref.flops)


@pytest.mark.parametrize("d", [4, 6, 8, 16, 24, 40])
@pytest.mark.parametrize("h_scale,c_scale,x_scale", [(1e-200, 1e200, 1e300), (1e-300, 1.0, 1.0), (1.0, 1.0, 1.0)])
def test_extreme_scales_take_the_ieee_division_path(solver, d, h_scale, c_scale, x_scale):
    """Box QPs scaled so the triangular-solve quotients leave the Markstein
    range (|q| > 2^958): H ~ 1e-200 with gradients ~ 1e200 (forward-solve
    quotients ~ 1e300), H ~ 1e-300 with gradients ~ 1 (backward-solve
    quotients ~ 1e300); both reach the PCG in the oracle.  The branch-free
    quotients flag it and the solve is recomputed with IEEE divisions
    (DESIGN.md §3).  Warp (d <= 16) and block (d = 24, 40) kernels, bitwise
    against the oracle; unscaled control case."""
    from paper_2106_14995_b200 import ProblemBatch

    b = synth.boxqp(48, d, seed=40 + d)
    params = b.params.copy()
    params[:, :d * d] *= h_scale
    params[:, d * d:] *= c_scale
    sb = ProblemBatch(b.family, d, b.lower * x_scale, b.upper * x_scale, np.ascontiguousarray(params),
                      b.x0 * x_scale)
    cfg = TronConfig(max_iter=25, tol_pg=1e-300)
    res = solver.solve_batch(sb, cfg=cfg, count_flops=True)
    ref = po.solve_batch(sb, cfg=cfg, impl="oracle", workers=8)
    assert_bitwise(res, ref, label=f"d={d} h={h_scale} c={c_scale}")
    assert np.array_equal(host(res.flops), ref.flops)


# ---------------------------------------------------------------- thread form
# n = 4 batches of >= 4,096 (branch) / 8,192 (ncvx) problems run one thread per
# problem (csrc/tron_thread.cuh); these pin it to the oracle and to the warp
# form (KernelForm.WARP), also on small batches forced through it
# (KernelForm.THREAD).


@pytest.mark.parametrize("fam,count", [("ncvx", 8192), ("ncvx", 16384), ("branch", 16384), ("branch", 20467)])
def test_thread_form_default_routing_bitwise(solver, monkeypatch, fam, count):
    b = synth.make(fam, count, 4)
    res = solver.solve_batch(b)  # >= 8,192 / 4,096 problems (whole batch, any chunking): thread form
    ref = po.solve_batch(b, impl="oracle", workers=os.cpu_count() or 8)
    assert_bitwise(res, ref, label=f"{fam}4 thread form")
    for form in (KernelForm.WARP,):
        with forced_form(solver, form):
            assert_bitwise(solver.solve_batch(b), ref, label=f"{fam}4 {form.name} form")
    import torch

    from paper_2106_14995_b200 import ProblemBatch, Solver

    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    db = ProblemBatch(b.family, 4, t(b.lower), t(b.upper), t(b.params), t(b.x0))
    out = Solver.alloc_result(count, 4, device=True)
    solver.solve_batch(db, out=out)  # device-resident: concurrent chunks of the same batch
    assert_bitwise(out, ref, label=f"{fam}4 thread form, device memspace")


@pytest.mark.parametrize("cfg", [TronConfig(), TronConfig(max_iter=1), TronConfig(delta0=0.3), TronConfig(tol_pg=1e-9),
                                 TronConfig(cg_tol=0.5, mu0=0.1, interp_factor=0.25),
                                 TronConfig(sigma1=0.1, sigma2=0.3, sigma3=2.0, eta0=0.01, delta_max=5.0)])
def test_thread_form_config_variants_bitwise(solver, cfg):
    with forced_form(solver, KernelForm.THREAD):
        for b in (synth.ncvx(300, 4, seed=9), synth.branch(300, 4, seed=9)):
            assert_bitwise(solver.solve_batch(b, cfg=cfg), po.solve_batch(b, cfg=cfg, impl="oracle"),
                           label=f"thread form {cfg}")


@pytest.mark.parametrize("form", ["THREAD", "WARP"])
def test_small_forms_outside_box_infinite_bounds_and_bad_bounds(solver, form):
    with forced_form(solver, KernelForm[form]):
        _outside_box_inf_bad_bounds(solver)


def _outside_box_inf_bad_bounds(solver):
    b = synth.ncvx(200, 4, seed=11)
    b.lower[::3, 1] = -np.inf
    b.upper[::4, 2] = np.inf
    x0 = b.x0 * 5.0
    res = solver.solve_batch(b, x0)
    assert_bitwise(res, po.solve_batch(b, x0, impl="oracle"), label="thread form outside/inf")
    xs = host(res.x_star)
    assert (xs >= b.lower).all() and (xs <= b.upper).all()
    b.lower[7, 0] = b.upper[7, 0] + 1.0
    with pytest.raises(ValueError, match="lower bound exceeds upper bound"):
        solver.solve_batch(b)


@pytest.mark.parametrize("form", ["THREAD", "WARP"])
def test_small_forms_ragged_counts_and_device_memspace(solver, form):
    with forced_form(solver, KernelForm[form]):
        _ragged_device(solver, form)


def _ragged_device(solver, form):
    import torch

    from paper_2106_14995_b200 import ProblemBatch, Solver

    for n in (1, 63, 64, 65, 129):
        b = synth.ncvx(n, 4, seed=20 + n)
        assert_bitwise(solver.solve_batch(b), po.solve_batch(b, impl="oracle"), label=f"{form} form n={n}")
    b = synth.branch(1000, 4, seed=3)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    db = ProblemBatch(b.family, 4, t(b.lower), t(b.upper), t(b.params), t(b.x0))
    out = Solver.alloc_result(1000, 4, device=True)
    solver.solve_batch(db, out=out)
    assert_bitwise(out, po.solve_batch(b, impl="oracle"), label=f"{form} form device memspace")
