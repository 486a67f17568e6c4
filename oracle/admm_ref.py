"""TEST INFRASTRUCTURE ONLY -- an independent restatement of the component
ADMM of SPEC.md:319-441 in numpy, written from the SPEC's formulas, NOT from
csrc/tb_admm.h / tb_admm_host.h (which both the device and
oracle/admm_oracle.c use).  It pins those shared closed forms independently:
the device's (and the C oracle's) residual trajectory must match this one
within the north star's tolerance (1e-6); it is not bit-identical (different
summation order, complex-arithmetic flows).

What it restates, each from the SPEC line cited:
* initial state: flat start v = 1, theta = 0, lambda = 0;
  rho0 for power couplings, 4 rho0 for voltage / angle couplings; initial
  consensus = the component values at the flat start (generator box midpoints);
* generator_update: box-projected proximal closed form;
* branch subproblems (Eq. (3)): solved by the C TRON
  restatement (oracle/tron_oracle.c) on the BRANCH family -- the problem
  definition itself is shared, the ADMM bookkeeping around it is not;
* bus_update: min sum_c rho_c/2 (x~_c - m_c)^2 subject to the
  P / Q balance rows of Eq. (2g)-(2h), m_c = x_c + lambda_c / rho_c; the
  voltage consensus w~ (a rho-weighted average of the adjacent copies) enters
  the rows through the shunt terms (-g_sh w on P, +b_sh w on Q; the design
  decision DESIGN.md records), so the rows are solved as one 2x2 KKT system;
  theta~ is the rho-weighted average;
* multiplier_update: lambda += rho (copy - consensus);
* residuals: primal max |copy - consensus|, dual
  max |rho (consensus_k - consensus_{k-1})|.
Flows are evaluated with complex arithmetic, S_ij = V_i conj(Y_ff V_i +
Y_ft V_j), S_ji = V_j conj(Y_tf V_i + Y_tt V_j) (SPEC.md:351-359 pi-model),
not through the family's real coefficient expressions."""
from __future__ import annotations

import numpy as np

from oracle import pyoracle

BRANCH = 3
NPARAMS = 36


class IndependentAdmm:
    def __init__(self, grid, rho_pq: float = 10.0, rho_va: float = 40.0, workers: int = 8):
        g = grid
        self.g = g
        self.workers = workers
        nb, ng, nl = g.n_bus, g.n_gen, g.n_branch
        c = np.asarray(g.br_coef, dtype=np.float64)
        self.Yff = c[:, 0] + 1j * c[:, 1]
        self.Yft = c[:, 2] + 1j * c[:, 3]
        self.Ytt = c[:, 4] + 1j * c[:, 5]
        self.Ytf = c[:, 6] + 1j * c[:, 7]
        self.fr = np.asarray(g.br_from, dtype=np.int64)
        self.to = np.asarray(g.br_to, dtype=np.int64)
        self.gb = np.asarray(g.gen_bus, dtype=np.int64)
        # branch component copies x = (v_i, v_j, th_i, th_j): flat start
        self.x = np.tile([1.0, 1.0, 0.0, 0.0], (nl, 1))
        # flow couplings (p_ij, q_ij, p_ji, q_ji): lambda, rho, consensus
        self.lam = np.zeros((nl, 4))
        self.rho = np.full((nl, 4), rho_pq)
        self.til = self.flows(self.x)
        # per branch end (i, j): w = v^2 and theta couplings
        self.lamw = np.zeros((nl, 2))
        self.rhow = np.full((nl, 2), rho_va)
        self.wtil = np.ones((nl, 2))
        self.lamt = np.zeros((nl, 2))
        self.rhot = np.full((nl, 2), rho_va)
        self.ttil = np.zeros((nl, 2))
        # generators: copies at the box midpoints, consensus = copies
        self.p = 0.5 * (g.gen_pmin + g.gen_pmax)
        self.q = 0.5 * (g.gen_qmin + g.gen_qmax)
        self.pt, self.qt = self.p.copy(), self.q.copy()
        self.lp, self.lq = np.zeros(ng), np.zeros(ng)
        self.rp, self.rq = np.full(ng, rho_pq), np.full(ng, rho_pq)
        self.wt, self.tt = np.ones(nb), np.zeros(nb)
        self.lo = np.stack([g.bus_vmin[self.fr], g.bus_vmin[self.to], np.full(nl, -2 * np.pi),
                            np.full(nl, -2 * np.pi)], axis=1)
        self.up = np.stack([g.bus_vmax[self.fr], g.bus_vmax[self.to], np.full(nl, 2 * np.pi),
                            np.full(nl, 2 * np.pi)], axis=1)
        self.history = []

    def flows(self, x):
        """(p_ij, q_ij, p_ji, q_ji) from the complex pi-model."""
        Vi = x[:, 0] * np.exp(1j * x[:, 2])
        Vj = x[:, 1] * np.exp(1j * x[:, 3])
        Sij = Vi * np.conj(self.Yff * Vi + self.Yft * Vj)
        Sji = Vj * np.conj(self.Ytf * Vi + self.Ytt * Vj)
        return np.stack([Sij.real, Sij.imag, Sji.real, Sji.imag], axis=1)

    def _branch_params(self):
        nl = self.g.n_branch
        prm = np.zeros((nl, NPARAMS))
        prm[:, 0:8] = self.g.br_coef
        prm[:, 8:12], prm[:, 12:16], prm[:, 16:20] = self.lam, self.rho, self.til
        prm[:, 20:22], prm[:, 22:24], prm[:, 24:26] = self.lamw, self.rhow, self.wtil
        prm[:, 26:28], prm[:, 28:30], prm[:, 30:32] = self.lamt, self.rhot, self.ttil
        return prm

    def step(self):
        g = self.g
        # generator_update: box-projected closed forms
        self.p = np.clip((self.rp * self.pt - self.lp - g.gen_c1) / (2.0 * g.gen_c2 + self.rp), g.gen_pmin, g.gen_pmax)
        self.q = np.clip((self.rq * self.qt - self.lq) / self.rq, g.gen_qmin, g.gen_qmax)
        # branch subproblems (Eq. (3)), warm started at the previous copies
        from paper_2106_14995_b200 import ProblemBatch

        b = ProblemBatch(BRANCH, 4, self.lo, self.up, self._branch_params(), self.x)
        r = pyoracle.solve_batch(b, impl="oracle", workers=self.workers)
        assert r.rc == 0, "branch subproblem raised"
        self.x = np.asarray(r.x_star, dtype=np.float64).reshape(-1, 4).copy()
        F = self.flows(self.x)
        # bus_update: m = copy + lambda / rho for every coupling at the bus
        nb = g.n_bus
        mp_g, mq_g = self.p + self.lp / self.rp, self.q + self.lq / self.rq
        mF = F + self.lam / self.rho  # [nl, 4]
        SP, SQ, WP, WQ = np.zeros(nb), np.zeros(nb), np.zeros(nb), np.zeros(nb)
        np.add.at(SP, self.gb, mp_g)
        np.add.at(SQ, self.gb, mq_g)
        np.add.at(WP, self.gb, 1.0 / self.rp)
        np.add.at(WQ, self.gb, 1.0 / self.rq)
        for end, bus in ((0, self.fr), (1, self.to)):  # flows leave the bus: coefficient -1
            np.add.at(SP, bus, -mF[:, 2 * end])
            np.add.at(SQ, bus, -mF[:, 2 * end + 1])
            np.add.at(WP, bus, 1.0 / self.rho[:, 2 * end])
            np.add.at(WQ, bus, 1.0 / self.rho[:, 2 * end + 1])
        v = self.x[:, 0:2]
        mw = v * v + self.lamw / self.rhow
        mt = self.x[:, 2:4] + self.lamt / self.rhot
        Sw, Rw, St, Rt = np.zeros(nb), np.zeros(nb), np.zeros(nb), np.zeros(nb)
        for end, bus in ((0, self.fr), (1, self.to)):
            np.add.at(Sw, bus, self.rhow[:, end] * mw[:, end])
            np.add.at(Rw, bus, self.rhow[:, end])
            np.add.at(St, bus, self.rhot[:, end] * mt[:, end])
            np.add.at(Rt, bus, self.rhot[:, end])
        aP, aQ = -np.asarray(g.bus_gsh, dtype=np.float64), np.asarray(g.bus_bsh, dtype=np.float64)
        wbar = Sw / Rw
        # KKT of  sum a_c x~_c + a_w w~ = rhs  for the P and Q rows, w~ = wbar - (aP muP + aQ muQ) / Rw
        A11, A22, A12 = WP + aP * aP / Rw, WQ + aQ * aQ / Rw, aP * aQ / Rw
        r1 = SP + aP * wbar - g.bus_pd
        r2 = SQ + aQ * wbar - g.bus_qd
        det = A11 * A22 - A12 * A12
        muP = (r1 * A22 - A12 * r2) / det
        muQ = (A11 * r2 - A12 * r1) / det
        wt = wbar - (aP * muP + aQ * muQ) / Rw
        tt = St / Rt
        # consensus values of every coupling
        pt = mp_g - muP[self.gb] / self.rp
        qt = mq_g - muQ[self.gb] / self.rq
        til = np.empty_like(F)
        for end, bus in ((0, self.fr), (1, self.to)):
            til[:, 2 * end] = mF[:, 2 * end] + muP[bus] / self.rho[:, 2 * end]
            til[:, 2 * end + 1] = mF[:, 2 * end + 1] + muQ[bus] / self.rho[:, 2 * end + 1]
        wtil = np.stack([wt[self.fr], wt[self.to]], axis=1)
        ttil = np.stack([tt[self.fr], tt[self.to]], axis=1)
        # residuals and multiplier_update
        gaps = [self.p - pt, self.q - qt, F - til, v * v - wtil, self.x[:, 2:4] - ttil]
        moves = [self.rp * (pt - self.pt), self.rq * (qt - self.qt), self.rho * (til - self.til),
                 self.rhow * (wtil - self.wtil), self.rhot * (ttil - self.ttil)]
        primal = max(float(np.max(np.abs(a))) if a.size else 0.0 for a in gaps)
        dual = max(float(np.max(np.abs(a))) if a.size else 0.0 for a in moves)
        self.lp += self.rp * gaps[0]
        self.lq += self.rq * gaps[1]
        self.lam += self.rho * gaps[2]
        self.lamw += self.rhow * gaps[3]
        self.lamt += self.rhot * gaps[4]
        self.pt, self.qt, self.til, self.wtil, self.ttil, self.wt, self.tt = pt, qt, til, wtil, ttil, wt, tt
        self.history.append((primal, dual))
        return primal, dual
