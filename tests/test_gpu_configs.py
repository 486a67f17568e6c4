"""The configurations VERDICT r1 found untested, on the GPU, bit for bit:

* C5 (BASELINE configs[4]): the 70,000-branch synthetic grid, ADMM at N = 1
  through the sharded driver, every iteration against the CPU oracle;
* the product's multi-partition paths on one GPU: a tb_context over devices
  (0, 0) (two partitions, batch.hpp:61-70) and two tb_admm shards of one
  grid in one process, the all-gather done by device copies;
* C3 (configs[2]) at its configured batch of 32,768 for d = 8 / 16 / 32 and on
  4,096-problem subsets at d = 64 / 128;
* a 50-iteration C4 (configs[3]) trajectory, through both the per-iteration
  step and the graph-replayed tb_admm_run;
* branch failures inside ADMM propagate."""
import os

import numpy as np
import pytest

from conftest import assert_bitwise, host
from oracle import pyoracle as po
from paper_2106_14995_b200 import EvaluationError, SingularFactorError, Solver, synth
from paper_2106_14995_b200 import admm as A

pytestmark = pytest.mark.gpu
W = os.cpu_count() or 8
STATE = (A.GEN_P, A.GEN_Q, A.GEN_PT, A.GEN_QT, A.GEN_LP, A.GEN_LQ, A.BUS_WT, A.BUS_TT, A.BRANCH_X, A.BRANCH_PARAMS,
         A.BRANCH_STATUS)


def c5_grid():
    nb = int(round(70000 * 13659 / 20467))  # C4's bus / branch ratio: 46,716 buses
    return synth.grid(nb, 70000, int(0.3 * nb))


def test_c5_grid_admm_bitwise_vs_oracle():
    g = c5_grid()
    assert (g.n_bus, g.n_branch, g.n_gen) == (46716, 70000, 14014)
    dev = A.ShardedAdmm(g, 0, 1, 0)  # the C5 driver at N = 1 (no collective)
    cpu = po.OracleAdmm(g, workers=W)
    for k in range(3):
        assert dev.step() == cpu.step(), f"C5 iteration {k}"
    for what in STATE:
        assert np.array_equal(dev.solver.get(what), cpu.get(what)), what


def test_c5_graph_run_with_ranked_stage_equals_steps():
    """C5's branch stage is ranked (beyond one wave); the order
    kernels are captured in tb_admm_run's CUDA graph.  The graph run and the
    blocking steps (bitwise = the oracle, above) must leave the same state."""
    g = c5_grid()
    a, b = A.AdmmSolver(g), A.AdmmSolver(g)
    try:
        steps = [a.step() for _ in range(4)]
        assert list(b.run(4, check_every=2)) == steps  # residual trajectory, bit for bit
        for what in STATE:
            assert np.array_equal(a.get(what), b.get(what)), what
    finally:
        a.close()
        b.close()


def test_multi_partition_context_on_one_gpu():
    """tb_solve_batch over a context of devices (0, 0): two partitions, each on
    its own stream, bit-identical to one partition; two partition times."""
    b = synth.branch(65536, 6, seed=2)
    one, two = Solver((0,)), Solver((0, 0))
    try:
        r1 = one.solve_batch(b)
        r2 = two.solve_batch(b)
        assert_bitwise(r2, r1, label="devices (0,0) vs (0,)")
        assert len(r2.partition_times) == 2 and min(r2.partition_times) > 0
        b3 = synth.ncvx(999, 40, seed=7)  # block kernel, ragged split (500 + 499)
        assert_bitwise(two.solve_batch(b3), po.solve_batch(b3, impl="oracle", workers=W), label="(0,0) block")
        assert_bitwise(Solver((0, 0, 0)).solve_batch(b3), po.solve_batch(b3, impl="oracle", workers=W),
                       label="(0,0,0) block")
    finally:
        one.close()
        two.close()


@pytest.mark.parametrize("line_limits", [False, True])
def test_two_admm_shards_in_one_process(line_limits):
    """Shards 0 and 1 of 2 of one grid on cuda:0, each with its own
    branch-solution buffer; the consensus exchange is done with device copies
    (what the NCCL all-gather does between processes).  Every iteration's
    residuals (max over the shards) and the state equal the single-shard run."""
    import torch

    g = synth.grid(900, 1301, 270, seed=17, shunt_frac=0.3)  # odd branch count: padded chunks
    opts = A.AdmmOptions(line_limits=line_limits)
    dim = opts.branch_dim
    world = 2
    chunk = (g.n_branch + world - 1) // world
    dev = torch.device("cuda", 0)
    xs = [torch.zeros((chunk * world, dim), dtype=torch.float64, device=dev) for _ in range(world)]
    res = [torch.zeros(3, dtype=torch.float64, device=dev) for _ in range(world)]
    shards = [A.AdmmSolver(g, opts, 0, r, world, x_buffer_ptr=xs[r].data_ptr()) for r in range(world)]
    ref = A.AdmmSolver(g, opts)
    st = torch.cuda.current_stream(dev).cuda_stream or 1
    for k in range(12):
        for s in shards:
            s.solve_components(st)
        for r in range(world):  # all-gather by copy: every buffer gets every shard's rows
            rows = slice(r * chunk, (r + 1) * chunk)
            for q in range(world):
                if q != r:
                    xs[q][rows].copy_(xs[r][rows])
        for r, s in enumerate(shards):
            s.update_consensus(st, res[r].data_ptr())
        got = torch.stack(res).max(dim=0).values.tolist()
        assert got[2] == -1.0
        assert (got[0], got[1]) == ref.step(), f"iteration {k}"
    for s in shards:
        for what in (A.BRANCH_X, A.BUS_WT, A.BUS_TT, A.GEN_P, A.GEN_LP):
            assert np.array_equal(s.get(what), ref.get(what)), what
    # branch parameters: lambda / rho / consensus columns are replicated on every
    # shard; the augmented-Lagrangian columns (mu, xi) of a branch live on the
    # shard that solves it, so the authoritative table takes each shard's rows
    full = np.concatenate([shards[r].get(A.BRANCH_PARAMS)[r * chunk:(r + 1) * chunk] for r in range(world)])
    assert np.array_equal(full, ref.get(A.BRANCH_PARAMS))


@pytest.mark.parametrize("d,count", [(8, 32768), (16, 32768), (32, 32768), (64, 4096), (128, 4096)])
def test_c3_configured_size_bitwise(solver, d, count):
    b = synth.ncvx(32768, d, seed=3 + d)  # the bench's C3 batch (seed 3 + d); subsets for d >= 64
    if count < b.count:
        from paper_2106_14995_b200 import ProblemBatch

        b = ProblemBatch(b.family, d, b.lower[:count], b.upper[:count], b.params[:count], b.x0[:count])
    res = solver.solve_batch(b)
    ref = po.solve_batch(b, impl="oracle", workers=W)
    assert_bitwise(res, ref, label=f"C3 d={d} x{count}")
    assert (host(res.status) <= 1).all()


def test_c4_fifty_iterations_bitwise_and_graph_run():
    g = synth.grid(13659, 20467, 4092)
    dev = A.AdmmSolver(g)
    cpu = po.OracleAdmm(g, workers=W)
    for k in range(50):
        assert dev.step() == cpu.step(), f"C4 iteration {k}"
    for what in STATE:
        assert np.array_equal(dev.get(what), cpu.get(what)), what
    # the same 50 iterations through tb_admm_run (one CUDA graph per
    # iteration, device stop flag, host poll every 16): same residuals, state
    run = A.AdmmSolver(g)
    hist = run.run(50, check_every=16)
    assert hist == dev.history
    for what in STATE:
        assert np.array_equal(run.get(what), dev.get(what)), what


def test_admm_run_stops_at_the_first_converged_iteration():
    g = synth.grid(300, 420, 90, seed=11, shunt_frac=0.3)
    steps = A.AdmmSolver(g)
    h = [steps.step() for _ in range(40)]
    tp, td = sorted(p for p, _ in h)[10], sorted(d for _, d in h)[25]
    k = next(i for i, (p, d) in enumerate(h) if p <= tp and d <= td)
    for every in (1, 7, 64):
        run = A.AdmmSolver(g)
        hist = run.run(40, tol_primal=tp, tol_dual=td, check_every=every)
        assert hist == h[:k + 1], every
        ref = A.AdmmSolver(g)
        for _ in range(k + 1):
            ref.step()
        assert np.array_equal(run.get(A.BRANCH_X), ref.get(A.BRANCH_X))
        assert np.array_equal(run.get(A.BUS_WT), ref.get(A.BUS_WT))


def test_admm_branch_failure_propagates():
    """a branch solve that throws in the reference is an error of
    the ADMM step -- in the single-process step, the graph run and the sharded
    driver -- naming the first failing branch.  Here bus 24 gets v_min > v_max,
    so its six branches have invalid bounds (tron.hpp:465-466, invalid_argument;
    status 6); the CPU oracle reports the same branches."""
    g = synth.grid(200, 260, 60, seed=3)
    g.bus_vmin = g.bus_vmin.copy()
    g.bus_vmin[24] = 1.2
    bad = np.nonzero((g.br_from == 24) | (g.br_to == 24))[0]
    assert bad[0] == 23
    s = A.AdmmSolver(g)
    with pytest.raises(ValueError, match="branch 23 failed with status 6"):
        s.step()
    st = s.get(A.BRANCH_STATUS)
    assert np.array_equal(np.nonzero(st)[0], bad) and (st[bad] == 6).all()
    with pytest.raises(ValueError, match="branch 23"):
        A.AdmmSolver(g).run(5)
    sh = A.ShardedAdmm(g, 0, 1, 0)
    with pytest.raises(Exception, match="branch 23"):
        sh.step()


def test_stage_times_and_sharded_partition_times():
    from paper_2106_14995_b200 import imbalance

    g = synth.grid(2000, 2800, 600, seed=5)
    s = A.AdmmSolver(g)
    s.step()
    comp, cons = s.stage_times()
    assert comp > 0 and cons > 0
    sh = A.ShardedAdmm(g, 0, 1, 0, record_times=True)
    for _ in range(4):
        sh.step()
    t = sh.partition_times()
    assert len(t) == 4 and all(len(r) == 1 and r[0] > 0 for r in t)
    st = imbalance([[r[0], 2 * r[0]] for r in t])  # two synthetic partitions: nu = (2/1.5 - 1) * 100
    assert abs(st.nu_max - 100.0 / 3.0) < 1e-9
