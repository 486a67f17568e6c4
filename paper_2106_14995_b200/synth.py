"""Synthetic problem batches with a portable counter-based RNG.

Every value is a pure function of (seed, problem index, draw index) through
splitmix64 -> (x >> 11) * 2^-53, so the same batch is produced on any host and
fed identically to the GPU and to the CPU oracle.
"""
from __future__ import annotations

import math

import numpy as np

from .tron import Family, ProblemBatch

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * _M1
    z = z ^ (z >> np.uint64(27))
    z = z * _M2
    return z ^ (z >> np.uint64(31))


class Stream:
    """Per-problem uniform streams: draw k of problem i is
    mix(base_i + (k+1) * golden), base_i = mix(seed * golden ^ (i+1))."""

    def __init__(self, seed: int, count: int, salt: int = 0):
        with np.errstate(over="ignore"):
            i = np.arange(1, count + 1, dtype=np.uint64)
            s = np.uint64((seed * 0x9E3779B97F4A7C15 + salt * 0xD1B54A32D192ED03) & 0xFFFFFFFFFFFFFFFF)
            self.base = _mix(s ^ _mix(i))
        self.k = 0

    def uniform(self, width: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
        """[count, width] uniforms in [lo, hi)."""
        with np.errstate(over="ignore"):
            ks = np.arange(self.k + 1, self.k + 1 + width, dtype=np.uint64)
            z = _mix(self.base[:, None] + ks[None, :] * _GOLDEN)
        self.k += width
        u = (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
        return lo + (hi - lo) * u


def ncvx(count: int, d: int, seed: int = 1) -> ProblemBatch:
    """f = 0.5 e'He + 0.25 sum k e^4 + sum a sin(x), e = x - c (tb_families.h NCVX).
    H_ij = H_ji ~ U(-1,1), c ~ 1.5 U(-1,1), k ~ U(0.5,1.5), a ~ 0.3 U(-1,1),
    l ~ -1 + 0.5 U(-1,1), u ~ 1 + 0.5 U(-1,1), x0 ~ 0.5 U(-1,1)."""
    st = Stream(seed, count, salt=d)
    npk = d * (d + 1) // 2
    Hp = st.uniform(npk, -1.0, 1.0)
    c = 1.5 * st.uniform(d, -1.0, 1.0)
    k = st.uniform(d, 0.5, 1.5)
    a = 0.3 * st.uniform(d, -1.0, 1.0)
    lo = -1.0 + 0.5 * st.uniform(d, -1.0, 1.0)
    up = 1.0 + 0.5 * st.uniform(d, -1.0, 1.0)
    x0 = 0.5 * st.uniform(d, -1.0, 1.0)
    params = np.ascontiguousarray(np.concatenate([Hp, c, k, a], axis=1))
    return ProblemBatch(Family.NCVX, d, lo, up, params, x0)


def boxqp(count: int, d: int, seed: int = 5, spd_boost: float = 0.5) -> ProblemBatch:
    """tests/unit/tron_test.cpp:196-212 shapes: H = B'B/n + 0.5 I (random_spd,
    tests/support/test_util.hpp:50-63), c ~ U(-2,2), l ~ U(-1,0),
    u = l + U(0.2,1.5), x0 ~ U(-1,1).  params = [H col-major | c]."""
    st = Stream(seed, count, salt=100 + d)
    B = st.uniform(d * d, -1.0, 1.0).reshape(count, d, d)
    H = np.einsum("bki,bkj->bij", B, B) / d + spd_boost * np.eye(d)[None]
    H = 0.5 * (H + np.transpose(H, (0, 2, 1)))
    c = st.uniform(d, -2.0, 2.0)
    lo = st.uniform(d, -1.0, 0.0)
    up = lo + st.uniform(d, 0.2, 1.5)
    x0 = st.uniform(d, -1.0, 1.0)
    Hcm = np.transpose(H, (0, 2, 1)).reshape(count, d * d)  # column-major
    params = np.ascontiguousarray(np.concatenate([Hcm, c], axis=1))
    return ProblemBatch(Family.BOXQP, d, lo, up, params, x0)


def hs45(count: int, d: int) -> ProblemBatch:
    """batch.hpp:116-131: l = 0, u_i = i (1-based), default start u/2."""
    up = np.tile(np.arange(1, d + 1, dtype=np.float64), (count, 1))
    lo = np.zeros_like(up)
    return ProblemBatch(Family.HS45, d, lo, up, None, 0.5 * up)


def pi_model(r, x, bc, tap, shift=None):
    """SPEC.md:351-359 / SURVEY App. C pi-model admittances -> the 8 flow
    coefficients (gff, bff, gft, bft, gtt, btt, gtf, btf)."""
    shift = np.zeros_like(r) if shift is None else shift
    z2 = r * r + x * x
    g, b = r / z2, -x / z2
    t2 = tap * tap
    cs, sn = np.cos(shift), np.sin(shift)
    # Y_ff = (y + j bc/2)/tap^2 ; Y_tt = y + j bc/2
    gff, bff = g / t2, (b + 0.5 * bc) / t2
    gtt, btt = g, b + 0.5 * bc
    # Y_ft = -y / conj(tau), Y_tf = -y / tau, tau = tap e^{j shift}
    # -y/conj(tau) = -(g+jb) e^{j shift}/tap ; -y/tau = -(g+jb) e^{-j shift}/tap
    gft, bft = -(g * cs - b * sn) / tap, -(g * sn + b * cs) / tap
    gtf, btf = -(g * cs + b * sn) / tap, -(b * cs - g * sn) / tap
    return np.stack([gff, bff, gft, bft, gtt, btt, gtf, btf], axis=-1)


def branch_flows(coef, vi, vj, ti, tj):
    """(p_ij, q_ij, p_ji, q_ji) of PAPER.md:542-545 (numpy libm trig; data
    generation only, never compared bitwise)."""
    gff, bff, gft, bft, gtt, btt, gtf, btf = [coef[..., k] for k in range(8)]
    wi, wj = vi * vi, vj * vj
    wr = vi * vj * np.cos(ti - tj)
    wim = vi * vj * np.sin(ti - tj)
    pij = gff * wi + gft * wr + bft * wim
    qij = -bff * wi - bft * wr + gft * wim
    pji = gtt * wj + gtf * wr - btf * wim
    qji = -btt * wj - btf * wr - gtf * wim
    return np.stack([pij, qij, pji, qji], axis=-1)


def branch(count: int, dim: int = 6, seed: int = 2, rho_p: float = 10.0, rho_v: float = 40.0) -> ProblemBatch:
    """Synthetic ADMM branch subproblems: dim 4 = Eq. (3),
    dim 6 = with line-limit slacks and augmented-Lagrangian terms."""
    assert dim in (4, 6)
    st = Stream(seed, count, salt=200 + dim)
    r = st.uniform(1, 0.001, 0.051)[:, 0]
    x = st.uniform(1, 0.01, 0.31)[:, 0]
    bc = st.uniform(1, 0.0, 0.1)[:, 0]
    tap = st.uniform(1, 0.975, 1.025)[:, 0]
    coef = pi_model(r, x, bc, tap)
    v = st.uniform(2, 0.95, 1.05)
    th = st.uniform(2, -0.1, 0.1)
    F = branch_flows(coef, v[:, 0], v[:, 1], th[:, 0], th[:, 1])
    Ft = F * (1.0 + 0.1 * st.uniform(4, -1.0, 1.0))
    wt = v * v * (1.0 + 0.1 * st.uniform(2, -1.0, 1.0))
    tt = th * (1.0 + 0.1 * st.uniform(2, -1.0, 1.0))
    lam = st.uniform(8, -1.0, 1.0)
    mu = st.uniform(2, 0.0, 1.0)
    smag = np.maximum(np.hypot(Ft[:, 0], Ft[:, 1]), np.hypot(Ft[:, 2], Ft[:, 3]))
    rate = smag * st.uniform(1, 0.9, 1.3)[:, 0]
    smax2 = rate * rate
    P = np.zeros((count, 36))
    P[:, 0:8] = coef
    P[:, 8:12] = lam[:, 0:4]
    P[:, 12:16] = rho_p
    P[:, 16:20] = Ft
    P[:, 20:22] = lam[:, 4:6]
    P[:, 22:24] = rho_v
    P[:, 24:26] = wt
    P[:, 26:28] = lam[:, 6:8]
    P[:, 28:30] = rho_v
    P[:, 30:32] = tt
    P[:, 32:34] = mu
    P[:, 34] = 10.0
    P[:, 35] = smax2
    lo = np.empty((count, dim))
    up = np.empty((count, dim))
    lo[:, 0:2], up[:, 0:2] = 0.9, 1.1
    lo[:, 2:4], up[:, 2:4] = -2.0 * math.pi, 2.0 * math.pi
    x0 = np.zeros((count, dim))
    x0[:, 0:2] = 1.0
    if dim == 6:
        lo[:, 4:6] = -smax2[:, None]
        up[:, 4:6] = 0.0
    return ProblemBatch(Family.BRANCH, dim, lo, up, np.ascontiguousarray(P), x0)


def make(family: str, count: int, dim: int, seed: int = None) -> ProblemBatch:
    if family == "ncvx":
        return ncvx(count, dim, seed if seed is not None else 1)
    if family == "boxqp":
        return boxqp(count, dim, seed if seed is not None else 5)
    if family == "hs45":
        return hs45(count, dim)
    if family in ("branch", "branch4", "branch6"):
        return branch(count, dim, seed if seed is not None else 2)
    raise ValueError(family)


# ------------------------------------------------------------------ ADMM grids
def grid(n_bus: int, n_branch: int, n_gen: int, seed: int = 4, load_factor: float = 0.6, shunt_frac: float = 0.1,
         rate: tuple = (0.5, 3.0)):
    """Synthetic AC-OPF network: random spanning tree plus
    extra edges up to n_branch, pi-model branches like C2, generators on
    random buses, loads at `load_factor` of generation capacity.  Returns an
    admm.Grid (per-unit)."""
    from .admm import Grid

    assert n_branch >= n_bus - 1 and n_bus >= 2
    rng = Stream(seed, 1, salt=900 + n_bus)
    u = lambda k, lo=0.0, hi=1.0: rng.uniform(k, lo, hi)[0]  # noqa: E731
    parent = np.floor(u(n_bus - 1) * np.arange(1, n_bus)).astype(np.int64)  # parent < child
    frm = [parent]
    to = [np.arange(1, n_bus)]
    extra = n_branch - (n_bus - 1)
    if extra > 0:
        a = np.floor(u(extra) * n_bus).astype(np.int64)
        b = np.floor(u(extra) * (n_bus - 1)).astype(np.int64)
        b = np.where(b >= a, b + 1, b)  # b != a
        frm.append(a)
        to.append(b)
    br_from = np.concatenate(frm).astype(np.int32)
    br_to = np.concatenate(to).astype(np.int32)
    r = u(n_branch, 0.001, 0.05)
    x = u(n_branch, 0.01, 0.3)
    bc = u(n_branch, 0.0, 0.1)
    tap = np.where(u(n_branch) < 0.2, u(n_branch, 0.95, 1.05), 1.0)
    coef = pi_model(r, x, bc, tap)
    gen_bus = np.sort(np.floor(u(n_gen) * n_bus).astype(np.int32))
    pmax = u(n_gen, 0.5, 5.0)
    w = u(n_bus, 0.0, 1.0)
    pd = load_factor * pmax.sum() * w / w.sum()
    qd = pd * u(n_bus, 0.1, 0.4)
    sh = u(n_bus) < shunt_frac
    smax = u(n_branch, rate[0], rate[1])  # line ratings s-bar (per unit), used with line limits on
    return Grid(
        bus_pd=pd, bus_qd=qd, bus_gsh=np.where(sh, u(n_bus, 0.0, 0.01), 0.0),
        bus_bsh=np.where(sh, u(n_bus, 0.0, 0.1), 0.0), bus_vmin=np.full(n_bus, 0.9), bus_vmax=np.full(n_bus, 1.1),
        gen_bus=gen_bus, gen_c2=u(n_gen, 0.005, 0.05), gen_c1=u(n_gen, 1.0, 10.0), gen_pmin=np.zeros(n_gen),
        gen_pmax=pmax, gen_qmin=-0.5 * pmax, gen_qmax=0.5 * pmax, br_from=br_from, br_to=br_to,
        br_coef=np.ascontiguousarray(coef), br_smax2=smax * smax)


def two_bus(pd: float = 0.5, qd: float = 0.1, r: float = 0.01, x: float = 0.1, smax: float = None):
    """SPEC.md:411 single-branch 2-bus toy: one generator at bus 0, one load at bus 1."""
    from .admm import Grid

    coef = pi_model(np.array([r]), np.array([x]), np.array([0.0]), np.array([1.0]))
    return Grid(bus_pd=np.array([0.0, pd]), bus_qd=np.array([0.0, qd]), bus_gsh=np.zeros(2), bus_bsh=np.zeros(2),
                bus_vmin=np.full(2, 0.9), bus_vmax=np.full(2, 1.1), gen_bus=np.array([0], np.int32),
                gen_c2=np.array([0.1]), gen_c1=np.array([1.0]), gen_pmin=np.array([0.0]), gen_pmax=np.array([2.0]),
                gen_qmin=np.array([-1.0]), gen_qmax=np.array([1.0]), br_from=np.array([0], np.int32),
                br_to=np.array([1], np.int32), br_coef=np.ascontiguousarray(coef),
                br_smax2=None if smax is None else np.array([smax * smax]))
