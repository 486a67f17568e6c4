"""ADMM AC-OPF: the spec's closed-form examples, bus-update
exactness against an independent KKT-QP oracle, the 2-bus toy against a full
NLP solve, and (GPU) the device pipeline against the CPU oracle bit-for-bit."""
import os

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2106_14995_b200 import admm as A
from paper_2106_14995_b200 import synth


# ------------------------------------------------------------ closed forms
def test_generator_update_spec_examples():
    """SPEC.md:374-377."""
    assert po.admm_gen_p(0.5, 0.0, 0.0, 2.0, 1.0, 0.0, 10.0) == pytest.approx(2.0 / 3.0, abs=1e-15)
    assert po.admm_gen_p(0.0, 0.0, 0.0, 3.0, 0.7, 0.0, 10.0) == pytest.approx(0.7, abs=1e-15)  # pure proximal
    assert po.admm_gen_p(0.0, 0.0, -100.0, 1.0, 1.0, 0.0, 10.0) == 10.0  # clamp at p-bar
    # brute-force 1-d minimisation of c2 p^2 + c1 p + lam (p - pt) + rho/2 (p - pt)^2 over the box
    rng = np.random.default_rng(0)
    for _ in range(50):
        c2, c1, lam, rho, pt = rng.uniform(0, 1), rng.uniform(-2, 2), rng.uniform(-2, 2), rng.uniform(0.5, 5), rng.uniform(-1, 3)
        p = po.admm_gen_p(c2, c1, lam, rho, pt, 0.0, 2.0)
        grid_ = np.linspace(0.0, 2.0, 200001)
        obj = c2 * grid_**2 + c1 * grid_ + lam * (grid_ - pt) + rho / 2 * (grid_ - pt) ** 2
        assert abs(p - grid_[np.argmin(obj)]) <= 2e-5


def _one_step(grid):
    a = po.OracleAdmm(grid)
    a.step()
    return a


def test_bus_balance_holds_exactly_after_update():
    """after the bus update the balance rows hold at the
    consensus values (to 1e-10)."""
    g = synth.grid(400, 560, 120, seed=3)
    a = _one_step(g)
    pt, qt = a.get(A.GEN_PT), a.get(A.GEN_QT)
    prm = a.get(A.BRANCH_PARAMS)
    wt = a.get(A.BUS_WT)
    P = np.zeros(g.n_bus)
    Q = np.zeros(g.n_bus)
    np.add.at(P, g.gen_bus, pt)
    np.add.at(Q, g.gen_bus, qt)
    np.add.at(P, g.br_from, -prm[:, 16])
    np.add.at(Q, g.br_from, -prm[:, 17])
    np.add.at(P, g.br_to, -prm[:, 18])
    np.add.at(Q, g.br_to, -prm[:, 19])
    P -= g.bus_gsh * wt
    Q += g.bus_bsh * wt
    assert np.max(np.abs(P - g.bus_pd)) <= 1e-10
    assert np.max(np.abs(Q - g.bus_qd)) <= 1e-10


def test_bus_update_matches_kkt_qp_oracle():
    """the closed form equals the equality-constrained QP solved
    by an independent dense KKT system (numpy), shunt buses included."""
    g = synth.grid(60, 90, 20, seed=5, shunt_frac=0.5)
    # state before the bus update: run one step, then redo the bus update by hand
    a = po.OracleAdmm(g)
    a.step()
    a.step()  # nonzero multipliers
    # snapshot component values and multipliers, then compare the next consensus
    x = a.get(A.BRANCH_X)
    prm = a.get(A.BRANCH_PARAMS)
    gp, gq, lp, lq = a.get(A.GEN_P), a.get(A.GEN_Q), a.get(A.GEN_LP), a.get(A.GEN_LQ)
    # rebuild the QP of every bus from the same snapshot the oracle will use: the
    # oracle's next step recomputes components first, so test on a frozen copy:
    F = synth.branch_flows(prm[:, :8], x[:, 0], x[:, 1], x[:, 2], x[:, 3])
    for b in range(g.n_bus):
        comps = []  # (a_P, a_Q, a_w, m, rho, kind)
        for k in np.nonzero(g.gen_bus == b)[0]:
            comps.append((1.0, 0.0, 0.0, gp[k] + lp[k] / 10.0, 10.0))
            comps.append((0.0, 1.0, 0.0, gq[k] + lq[k] / 10.0, 10.0))
        rw, mw = [], []
        for l in np.nonzero(g.br_from == b)[0]:
            comps.append((-1.0, 0.0, 0.0, F[l, 0] + prm[l, 8] / prm[l, 12], prm[l, 12]))
            comps.append((0.0, -1.0, 0.0, F[l, 1] + prm[l, 9] / prm[l, 13], prm[l, 13]))
            rw.append(prm[l, 22]); mw.append(x[l, 0] ** 2 + prm[l, 20] / prm[l, 22])
        for l in np.nonzero(g.br_to == b)[0]:
            comps.append((-1.0, 0.0, 0.0, F[l, 2] + prm[l, 10] / prm[l, 14], prm[l, 14]))
            comps.append((0.0, -1.0, 0.0, F[l, 3] + prm[l, 11] / prm[l, 15], prm[l, 15]))
            rw.append(prm[l, 23]); mw.append(x[l, 1] ** 2 + prm[l, 21] / prm[l, 23])
        # one shared w variable with its copies as separate objective terms
        n = len(comps) + 1
        H = np.zeros((n, n)); c = np.zeros(n); Aeq = np.zeros((2, n))
        for i, (aP, aQ, _, m, r) in enumerate(comps):
            H[i, i] = r; c[i] = r * m; Aeq[0, i] = aP; Aeq[1, i] = aQ
        H[-1, -1] = sum(rw); c[-1] = sum(r * m for r, m in zip(rw, mw))
        Aeq[0, -1] = -g.bus_gsh[b]; Aeq[1, -1] = g.bus_bsh[b]
        K = np.block([[H, Aeq.T], [Aeq, np.zeros((2, 2))]])
        sol = np.linalg.solve(K, np.concatenate([c, [g.bus_pd[b], g.bus_qd[b]]]))
        xt = sol[:n]
        # closed form (the formula of tb_admm.h) in numpy
        SP = sum(aP * m for aP, aQ, _, m, r in comps if aP); WP = sum(1 / r for aP, aQ, _, m, r in comps if aP)
        SQ = sum(aQ * m for aP, aQ, _, m, r in comps if aQ); WQ = sum(1 / r for aP, aQ, _, m, r in comps if aQ)
        Rw = sum(rw); mbar = sum(r * m for r, m in zip(rw, mw)) / Rw
        aPw, aQw = -g.bus_gsh[b], g.bus_bsh[b]
        A11, A22, A12 = WP + aPw**2 / Rw, WQ + aQw**2 / Rw, aPw * aQw / Rw
        r1, r2 = SP + aPw * mbar - g.bus_pd[b], SQ + aQw * mbar - g.bus_qd[b]
        muP, muQ = np.linalg.solve([[A11, A12], [A12, A22]], [r1, r2])
        closed = [m - (aP * muP + aQ * muQ) / r for aP, aQ, _, m, r in comps] + [mbar - (aPw * muP + aQw * muQ) / Rw]
        assert np.max(np.abs(np.array(closed) - xt)) <= 1e-9 * max(1.0, np.max(np.abs(xt)))


def test_angle_consensus_and_multiplier_examples():
    """SPEC.md:386 (theta~ = 0.2 from copies 0.1, 0.3 with equal rho) and
    SPEC.md:393-395 (lambda = rho * gap) on a 2-bus network."""
    g = synth.two_bus()
    a = po.OracleAdmm(g)
    a.step()
    x = a.get(A.BRANCH_X)
    prm = a.get(A.BRANCH_PARAMS)
    tt = a.get(A.BUS_TT)
    # bus 0 has one angle copy (th_i of the branch): th~_0 = th_i + lambda/rho with lambda = 0
    assert tt[0] == x[0, 2]
    # after the step lambda_theta = rho (th - th~) = 0 at a single-copy bus
    assert prm[0, 26] == 0.0
    # generator multipliers moved by rho * (p - p~)
    lp = a.get(A.GEN_LP)
    assert abs(lp[0] - 10.0 * (a.get(A.GEN_P)[0] - a.get(A.GEN_PT)[0])) <= 1e-12


def test_two_bus_toy_converges_and_matches_full_nlp():
    """SPEC.md:411 / acceptance 6(a): primal residual <= 1e-5 and dispatch
    within 1e-3 p.u. of a direct full-NLP solve (scipy SLSQP, 6 variables)."""
    from scipy.optimize import minimize

    g = synth.two_bus()
    a = po.OracleAdmm(g)
    for _ in range(3000):
        p, d = a.step()
        if p <= 1e-6 and d <= 1e-3:
            break
    assert p <= 1e-5
    pg, qg = a.get(A.GEN_P)[0], a.get(A.GEN_Q)[0]
    cf = g.br_coef[0]

    def flows(z):
        vi, vj, ti, tj = z[2:6]
        return synth.branch_flows(cf, vi, vj, ti, tj)

    cons = [
        {"type": "eq", "fun": lambda z: z[0] - flows(z)[0]},             # bus 0: pg = p_ij
        {"type": "eq", "fun": lambda z: z[1] - flows(z)[1]},             # bus 0: qg = q_ij
        {"type": "eq", "fun": lambda z: -g.bus_pd[1] - flows(z)[2]},     # bus 1: -pd = p_ji
        {"type": "eq", "fun": lambda z: -g.bus_qd[1] - flows(z)[3]},
        {"type": "eq", "fun": lambda z: z[4]},                           # reference angle
    ]
    res = minimize(lambda z: g.gen_c2[0] * z[0] ** 2 + g.gen_c1[0] * z[0], x0=[0.5, 0.1, 1, 1, 0, 0],
                   bounds=[(0, 2), (-1, 1), (0.9, 1.1), (0.9, 1.1), (-6.3, 6.3), (-6.3, 6.3)],
                   constraints=cons, method="SLSQP", options={"ftol": 1e-14, "maxiter": 500})
    assert res.success
    # active dispatch (the cost depends on p only; q and v are not unique)
    assert abs(pg - res.x[0]) <= 1e-3
    assert abs(a.get(A.COST)[0] - res.fun) <= 1e-3 * abs(res.fun)
    assert -1.0 <= qg <= 1.0


# ------------------------------------------------------------ line limits
def _binding_grid():
    """A synthetic grid whose ratings bind: the d=4 (unlimited) ADMM flows
    after 40 iterations, with s-bar = 0.7 |S| on the 15 % most loaded lines."""
    g = synth.grid(150, 210, 40, seed=9, shunt_frac=0.3)
    a = po.OracleAdmm(g)
    for _ in range(40):
        a.step()
    x = a.get(A.BRANCH_X)
    s = np.array([max(np.hypot(*synth.branch_flows(g.br_coef[l], *x[l])[0:2]),
                      np.hypot(*synth.branch_flows(g.br_coef[l], *x[l])[2:4])) for l in range(g.n_branch)])
    cut = np.quantile(s, 0.85)
    g.br_smax2 = np.where(s >= cut, (0.7 * s) ** 2, 100.0)
    return g, s >= cut


def test_line_limits_enforced_by_auglag_loop():
    """with line_limits the branch stage is the d=6
    augmented-Lagrangian loop; the binding lines end feasible (|S| <= s-bar up
    to the AL tolerance), the slacks stay in their boxes, and mu moved only on
    the binding lines."""
    g, bind = _binding_grid()
    a = po.OracleAdmm(g, A.AdmmOptions(line_limits=True))
    for _ in range(60):
        a.step()
    x = a.get(A.BRANCH_X)
    assert x.shape == (g.n_branch, 6)
    assert a.get(A.LINE_VIOL)[0] <= 1e-5
    assert a.get(A.AUGLAG_ROUNDS)[0] > 60  # more than one round in some iterations
    for l in range(g.n_branch):
        f = synth.branch_flows(g.br_coef[l], *x[l, :4])
        for e in range(2):
            assert np.hypot(f[2 * e], f[2 * e + 1]) ** 2 <= g.br_smax2[l] + 1e-5
            assert -g.br_smax2[l] <= x[l, 4 + e] <= 0.0
    mu = a.get(A.BRANCH_PARAMS)[:, 32:34]
    assert np.abs(mu[bind]).max() > 0.0
    assert np.abs(mu[~bind]).max() < np.abs(mu[bind]).max()


def test_line_limits_off_is_the_d4_spec_path():
    """line_limits=False keeps the SPEC's 4-dimensional branch subproblem:
    the ratings are ignored and no AL round runs."""
    g = synth.grid(60, 80, 15, seed=3)
    a, b = po.OracleAdmm(g), po.OracleAdmm(g, A.AdmmOptions(line_limits=False))
    g.br_smax2 = None
    c = po.OracleAdmm(g)
    for _ in range(5):
        assert a.step() == b.step() == c.step()
    assert a.get(A.AUGLAG_ROUNDS)[0] == 0
    assert a.get(A.BRANCH_X).shape == (g.n_branch, 4)


# ------------------------------------------------------------ device
@pytest.mark.gpu
def test_device_admm_trajectory_bitwise_vs_oracle():
    """Every iteration's residuals and the full state equal the CPU oracle's
    bit for bit (the branch stage is exact TRON, the closed forms are shared)."""
    g = synth.grid(300, 420, 90, seed=11, shunt_frac=0.3)
    dev = A.AdmmSolver(g)
    cpu = po.OracleAdmm(g, workers=8)
    for k in range(25):
        assert dev.step() == cpu.step(), f"iteration {k}"
    for what in (A.GEN_P, A.GEN_Q, A.GEN_PT, A.GEN_QT, A.GEN_LP, A.GEN_LQ, A.BUS_WT, A.BUS_TT, A.BRANCH_X,
                 A.BRANCH_PARAMS, A.BRANCH_STATUS, A.COST):
        assert np.array_equal(dev.get(what), cpu.get(what)), what


@pytest.mark.gpu
def test_device_admm_c4_first_iterations_bitwise():
    """C4 shape (13,659 buses / 20,467 branches / 4,092 generators)."""
    g = synth.grid(13659, 20467, 4092)
    dev = A.AdmmSolver(g)
    cpu = po.OracleAdmm(g, workers=16)
    for k in range(3):
        assert dev.step() == cpu.step(), f"iteration {k}"
    assert np.array_equal(dev.get(A.BRANCH_PARAMS), cpu.get(A.BRANCH_PARAMS))


@pytest.fixture(scope="module")
def nccl_world1():
    """A world-size-1 NCCL group for the sharded-driver tests, torn down after them."""
    import os

    import torch.distributed as dist

    created = False
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1)
        created = True
    yield
    if created:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_path_world1_equals_single(nccl_world1):
    """The torch.distributed driver (C5 path) at world size 1 == AdmmSolver."""
    g = synth.grid(500, 700, 150, seed=2)
    sh = A.ShardedAdmm(g, 0, 1, 0)
    ref = A.AdmmSolver(g)
    for k in range(10):
        assert sh.step() == ref.step(), k
    assert np.array_equal(sh.solver.get(A.BRANCH_X), ref.get(A.BRANCH_X))


@pytest.mark.gpu
def test_device_admm_line_limits_bitwise_vs_oracle():
    """The d=6 augmented-Lagrangian branch stage on the device (compaction of
    the active branches, TRON, AL update kernel) against the oracle's loop:
    residuals, every state array, the AL round count and the line violation
    bit for bit."""
    g, _ = _binding_grid()
    opts = A.AdmmOptions(line_limits=True)
    dev = A.AdmmSolver(g, opts)
    cpu = po.OracleAdmm(g, opts, workers=8)
    for k in range(20):
        assert dev.step() == cpu.step(), f"iteration {k}"
    for what in (A.GEN_P, A.GEN_Q, A.BUS_WT, A.BUS_TT, A.BRANCH_X, A.BRANCH_PARAMS, A.BRANCH_STATUS, A.COST,
                 A.AUGLAG_ROUNDS, A.LINE_VIOL):
        assert np.array_equal(dev.get(what), cpu.get(what)), what


@pytest.mark.gpu
def test_sharded_path_world1_line_limits_equals_single(nccl_world1):
    """The torch.distributed driver with the d=6 branch stage (x rows of 6)."""
    g, _ = _binding_grid()
    opts = A.AdmmOptions(line_limits=True)
    sh = A.ShardedAdmm(g, 0, 1, 0, opts)
    ref = A.AdmmSolver(g, opts)
    for k in range(8):
        assert sh.step() == ref.step(), k
    assert np.array_equal(sh.solver.get(A.BRANCH_X), ref.get(A.BRANCH_X))
    assert sh.x.shape[1] == 6


@pytest.mark.gpu
def test_get_after_stages_on_caller_stream_sees_their_results():
    """tb_admm_get waits for the caller stream the stages were enqueued on (no
    host sync in between), and the entry points leave the current device alone."""
    import torch

    g = synth.grid(400, 560, 120, seed=5)
    dev = A.AdmmSolver(g)
    ref = A.AdmmSolver(g)
    s = torch.cuda.Stream()
    before = torch.cuda.current_device()
    for k in range(4):
        ref.step()
        dev.solve_components(s.cuda_stream)
        dev.update_consensus(s.cuda_stream)
        # no synchronisation here: get must order itself after stream s
        assert np.array_equal(dev.get(A.BRANCH_X), ref.get(A.BRANCH_X)), k
        assert np.array_equal(dev.get(A.BUS_WT), ref.get(A.BUS_WT)), k
    assert torch.cuda.current_device() == before


@pytest.mark.gpu
def test_thread_and_warp_branch_stage_forms_agree_bitwise():
    """The d = 4 branch stage runs one thread per branch, fused with the
    generator updates, by default (csrc/tron_thread.cuh) and the warp kernel
    with branch_form="warp"; both are bit-identical to the oracle, hence to
    each other (residuals every iteration and the state after 12)."""
    g = synth.grid(800, 1100, 240, seed=9, shunt_frac=0.3)
    t = A.AdmmSolver(g)
    w = A.AdmmSolver(g, A.AdmmOptions(branch_form="warp"))
    for k in range(12):
        assert t.step() == w.step(), k
    for what in (A.BRANCH_X, A.BRANCH_PARAMS, A.BUS_WT, A.GEN_P, A.GEN_LP):
        assert np.array_equal(t.get(what), w.get(what)), what


# ------------------------------------------- independent restatement (admm_ref)
def _rel(a, b):
    return max(abs(a[0] - b[0]) / max(abs(a[0]), 1e-300), abs(a[1] - b[1]) / max(abs(a[1]), 1e-300))


@pytest.mark.parametrize("which", ["synth", "case9"])
def test_oracle_admm_matches_independent_restatement(which):
    """oracle/admm_oracle.c shares its closed forms with the device
    (csrc/tb_admm.h); oracle/admm_ref.py restates SPEC.md:369-404 independently
    (numpy, complex-arithmetic flows, its own bus KKT).  Residual trajectories
    agree within the north star's 1e-6 (observed ~6e-8 after 40 iterations)."""
    import os

    from oracle.admm_ref import IndependentAdmm
    from paper_2106_14995_b200 import matpower

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    g = (synth.grid(300, 420, 90, seed=11, shunt_frac=0.3) if which == "synth"
         else matpower.load(os.path.join(root, "tests", "data", "case9.m")).grid)
    a, b = po.OracleAdmm(g, workers=8), IndependentAdmm(g)
    for k in range(40):
        ra, rb = a.step(), b.step()
        assert _rel(ra, rb) <= 1e-6, (k, ra, rb)
    assert np.max(np.abs(a.get(A.BUS_WT) - b.wt)) <= 1e-6
    assert np.max(np.abs(a.get(A.GEN_P) - b.p)) <= 1e-6


@pytest.mark.gpu
def test_device_admm_c4_matches_independent_restatement():
    """The device trajectory on C4 against the independent restatement."""
    from oracle.admm_ref import IndependentAdmm

    g = synth.grid(13659, 20467, 4092)
    dev, ind = A.AdmmSolver(g), IndependentAdmm(g, workers=16)
    worst = 0.0
    for k in range(15):
        r = _rel(dev.step(), ind.step())
        worst = max(worst, r)
        assert r <= 1e-6, (k, r)
    print(f"C4 device vs independent restatement: max relative residual difference {worst:.2e}")


@pytest.mark.gpu
def test_ranked_line_limit_stage_bitwise_vs_oracle():
    """Beyond one wave of warps the fused augmented-Lagrangian stage is
    launched in rank order (start projected gradient); the
    trajectory and the state stay the oracle's bit for bit."""
    g = synth.grid(4200, 6300, 1260, seed=21, shunt_frac=0.3, rate=(0.05, 0.6))
    opts = A.AdmmOptions(line_limits=True)
    dev = A.AdmmSolver(g, opts)
    cpu = po.OracleAdmm(g, opts, workers=os.cpu_count() or 8)
    try:
        for k in range(4):
            assert dev.step() == cpu.step(), f"iteration {k}"
        for what in (A.BRANCH_X, A.BRANCH_PARAMS, A.AUGLAG_ROUNDS, A.LINE_VIOL, A.BUS_WT):
            assert np.array_equal(dev.get(what), cpu.get(what)), what
    finally:
        dev.close()
        cpu.close()
