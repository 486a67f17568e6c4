/*
 * tb_admm.h — component ADMM for AC optimal power flow (SPEC.md:319-441,
 * PAPER.md:530-590), the consumer of the batched TRON path.  The reference
 * ships no code for it; this is the spec restated as plain C shared by the
 * device kernels (admm.cu) and the CPU oracle (oracle/admm_oracle.c), so
 * both produce identical bits for the same iteration.
 *
 * Couplings (component copy x  ==  bus-side consensus x~), each with its own
 * multiplier lambda and penalty rho:
 *   generator g at bus b : p_g, q_g                          (2)
 *   branch l = (i -> j)  : p_ij, q_ij at bus i, p_ji, q_ji at bus j (flows of
 *                          Eq. (2i)-(2l) at the branch's own voltages),
 *                          w_i = v_i^2, th_i at bus i, w_j, th_j at bus j   (8)
 * One ADMM iteration:
 *   1. generator update (closed form) and branch update
 *      (TRON on Eq. (3), warm start) — independent, may run concurrently
 *   2. bus update (closed form): per bus minimise
 *      sum_c rho_c/2 (x~_c - m_c)^2, m_c = x_c + lambda_c / rho_c, subject to
 *      the balance rows (Eq. 2g-2h)
 *          sum p~_g - sum p~_l - gsh w~ = pd ,  sum q~_g - sum q~_l + bsh w~ = qd
 *      where w~ aggregates the voltage copies (one shared variable with weight
 *      R_w = sum rho_w and target sum rho_w m_w / R_w).  The two rows share
 *      only w~ (through the shunt), so the KKT system is 2x2; without a shunt
 *      it is the SPEC's one-multiplier-per-row closed form.  th~ is the
 *      rho-weighted average of the angle copies (no balance row).
 *   3. multipliers lambda += rho (x - x~)
 *   4. residuals primal = max |x - x~|, dual = max |rho (x~_k - x~_{k-1})|
 *
 * Every coupling belongs to exactly one bus, so steps 2-4 are one pass per bus
 * with no write conflicts.  Branch couplings keep lambda / rho / x~ inside the
 * branch family's parameter rows (TB_BR_* in tb_families.h), which the TRON
 * kernel reads directly.
 */
#ifndef TB_ADMM_H
#define TB_ADMM_H

#include <stdint.h>

#include "tb_families.h"

/* All arrays in one memory space (host for the oracle, device for kernels). */
typedef struct tb_admm_view {
    int32_t n_bus, n_gen, n_branch, branch_dim;
    /* buses */
    const double *bus_pd, *bus_qd, *bus_gsh, *bus_bsh;
    double *bus_wt, *bus_tt; /* consensus w~, th~ */
    /* generators */
    const int32_t* gen_bus;
    const double *gen_c2, *gen_c1, *gen_pmin, *gen_pmax, *gen_qmin, *gen_qmax;
    double *gen_p, *gen_q;   /* component copies */
    double *gen_lp, *gen_lq; /* multipliers */
    double *gen_rp, *gen_rq; /* penalties */
    double *gen_pt, *gen_qt; /* consensus p~, q~ */
    /* branches: x [n_branch][branch_dim] = (v_i, v_j, th_i, th_j[, s_ij, s_ji]) */
    const int32_t *br_from, *br_to;
    double* br_params; /* [n_branch][TB_BR_NPARAMS] */
    const double* br_x;
    /* CSR incidence by bus, in canonical order: generators (ascending index),
     * then branch ends (ascending branch, end 0 = from, 1 = to) */
    const int32_t *gen_ptr, *gen_idx; /* [n_bus + 1], [n_gen] */
    const int32_t *end_ptr, *end_idx; /* [n_bus + 1], [2 n_branch], value 2 * l + end */
} tb_admm_view;

/* p = P[(rho p~ - lambda - c1) / (2 c2 + rho)], q = P[(rho q~ - lambda) / rho] */
TB_HD void tb_admm_gen_update(const tb_admm_view* v, int g) {
    const double rp = v->gen_rp[g], rq = v->gen_rq[g];
    const double p = (rp * v->gen_pt[g] - v->gen_lp[g] - v->gen_c1[g]) / (2.0 * v->gen_c2[g] + rp);
    const double q = (rq * v->gen_qt[g] - v->gen_lq[g]) / rq;
    v->gen_p[g] = tb_smin(tb_smax(p, v->gen_pmin[g]), v->gen_pmax[g]);
    v->gen_q[g] = tb_smin(tb_smax(q, v->gen_qmin[g]), v->gen_qmax[g]);
}

/* flow f (0 p_ij, 1 q_ij, 2 p_ji, 3 q_ji) at the branch's voltages: the same
 * expression the BRANCH family's objective uses (tb_br_flow). */
TB_HD double tb_admm_flow(const double* base, const double* prm, int f) {
    double fa, fb, fc;
    tb_br_coef(f, prm, &fa, &fb, &fc);
    const double w_own = f < 2 ? base[TB_BRB_WII] : base[TB_BRB_WJJ];
    return (fa * w_own + fb * base[TB_BRB_WR]) + fc * base[TB_BRB_WI];
}

typedef struct {
    double primal, dual;
} tb_admm_res;

TB_HD double tb_admm_absd(double a) { return a < 0.0 ? -a : a; }

/* One bus: consensus, multipliers and residual terms of all its couplings. */
TB_HD void tb_admm_bus_update(const tb_admm_view* v, int b, tb_admm_res* res) {
    const double pd = v->bus_pd[b], qd = v->bus_qd[b];
    const double aPw = -v->bus_gsh[b], aQw = v->bus_bsh[b];
    const int D = v->branch_dim;
    double SP = 0.0, WP = 0.0, SQ = 0.0, WQ = 0.0, Sw = 0.0, Rw = 0.0, St = 0.0, Rt = 0.0;
    /* pass 1: sums in canonical CSR order */
    for (int k = v->gen_ptr[b]; k < v->gen_ptr[b + 1]; ++k) {
        const int g = v->gen_idx[k];
        SP += v->gen_p[g] + v->gen_lp[g] / v->gen_rp[g];
        WP += 1.0 / v->gen_rp[g];
        SQ += v->gen_q[g] + v->gen_lq[g] / v->gen_rq[g];
        WQ += 1.0 / v->gen_rq[g];
    }
    for (int k = v->end_ptr[b]; k < v->end_ptr[b + 1]; ++k) {
        const int e = v->end_idx[k], l = e >> 1, end = e & 1;
        const double* prm = v->br_params + (long)l * TB_BR_NPARAMS;
        const double* x = v->br_x + (long)l * D;
        double base[8];
        tb_br_base(x, base);
        const int fp = 2 * end, fq = 2 * end + 1;
        SP -= tb_admm_flow(base, prm, fp) + prm[TB_BR_LAM + fp] / prm[TB_BR_RHO + fp];
        WP += 1.0 / prm[TB_BR_RHO + fp];
        SQ -= tb_admm_flow(base, prm, fq) + prm[TB_BR_LAM + fq] / prm[TB_BR_RHO + fq];
        WQ += 1.0 / prm[TB_BR_RHO + fq];
        const double vv = x[end];
        const double rw = prm[TB_BR_RHOW + end], rt = prm[TB_BR_RHOT + end];
        Sw += rw * (vv * vv + prm[TB_BR_LAMW + end] / rw);
        Rw += rw;
        St += rt * (x[2 + end] + prm[TB_BR_LAMT + end] / rt);
        Rt += rt;
    }
    const double mbar = Sw / Rw;
    const double r1 = (SP + aPw * mbar) - pd;
    const double r2 = (SQ + aQw * mbar) - qd;
    const double A12 = (aPw * aQw) / Rw;
    double muP, muQ;
    if (A12 == 0.0) {
        muP = r1 / (WP + (aPw * aPw) / Rw);
        muQ = r2 / (WQ + (aQw * aQw) / Rw);
    } else {
        const double A11 = WP + (aPw * aPw) / Rw, A22 = WQ + (aQw * aQw) / Rw;
        const double det = A11 * A22 - A12 * A12;
        muP = (r1 * A22 - A12 * r2) / det;
        muQ = (A11 * r2 - A12 * r1) / det;
    }
    const double wt = mbar - (aPw * muP + aQw * muQ) / Rw;
    const double tt = St / Rt;
    /* pass 2: consensus, multipliers, residuals */
    double pr = 0.0, du = 0.0;
#define TB_ADMM_COUPLING(X, XT_OLD, XT_NEW, RHO, LAM_REF)                    \
    do {                                                                     \
        const double d_ = tb_admm_absd((RHO) * ((XT_NEW) - (XT_OLD)));      \
        if (du < d_) du = d_;                                                \
        const double g_ = (X) - (XT_NEW);                                    \
        if (pr < tb_admm_absd(g_)) pr = tb_admm_absd(g_);                    \
        LAM_REF += (RHO) * g_;                                               \
    } while (0)
    for (int k = v->gen_ptr[b]; k < v->gen_ptr[b + 1]; ++k) {
        const int g = v->gen_idx[k];
        const double rp = v->gen_rp[g], rq = v->gen_rq[g];
        const double ptn = (v->gen_p[g] + v->gen_lp[g] / rp) - muP / rp;
        const double qtn = (v->gen_q[g] + v->gen_lq[g] / rq) - muQ / rq;
        TB_ADMM_COUPLING(v->gen_p[g], v->gen_pt[g], ptn, rp, v->gen_lp[g]);
        TB_ADMM_COUPLING(v->gen_q[g], v->gen_qt[g], qtn, rq, v->gen_lq[g]);
        v->gen_pt[g] = ptn;
        v->gen_qt[g] = qtn;
    }
    for (int k = v->end_ptr[b]; k < v->end_ptr[b + 1]; ++k) {
        const int e = v->end_idx[k], l = e >> 1, end = e & 1;
        double* prm = v->br_params + (long)l * TB_BR_NPARAMS;
        const double* x = v->br_x + (long)l * D;
        double base[8];
        tb_br_base(x, base);
        const int fp = 2 * end, fq = 2 * end + 1;
        const double Fp = tb_admm_flow(base, prm, fp), Fq = tb_admm_flow(base, prm, fq);
        const double rP = prm[TB_BR_RHO + fp], rQ = prm[TB_BR_RHO + fq];
        const double Ftp = (Fp + prm[TB_BR_LAM + fp] / rP) + muP / rP;
        const double Ftq = (Fq + prm[TB_BR_LAM + fq] / rQ) + muQ / rQ;
        TB_ADMM_COUPLING(Fp, prm[TB_BR_TIL + fp], Ftp, rP, prm[TB_BR_LAM + fp]);
        TB_ADMM_COUPLING(Fq, prm[TB_BR_TIL + fq], Ftq, rQ, prm[TB_BR_LAM + fq]);
        prm[TB_BR_TIL + fp] = Ftp;
        prm[TB_BR_TIL + fq] = Ftq;
        const double vv = x[end];
        TB_ADMM_COUPLING(vv * vv, prm[TB_BR_WTIL + end], wt, prm[TB_BR_RHOW + end], prm[TB_BR_LAMW + end]);
        TB_ADMM_COUPLING(x[2 + end], prm[TB_BR_TTIL + end], tt, prm[TB_BR_RHOT + end], prm[TB_BR_LAMT + end]);
        prm[TB_BR_WTIL + end] = wt;
        prm[TB_BR_TTIL + end] = tt;
    }
#undef TB_ADMM_COUPLING
    v->bus_wt[b] = wt;
    v->bus_tt[b] = tt;
    res->primal = pr;
    res->dual = du;
}

/* ---- line limits (options.line_limits, branch dim 6) ------------------
 * h_l = p_l^2 + q_l^2 + s_l at the branch solution x, line end l (0 = from,
 * 1 = to), with the BRANCH family's own flow expressions (tb_br_line). */
TB_HD double tb_admm_line_hmax(const double* x, const double* prm, double* h) {
    double base[8];
    tb_br_base(x, base);
    double hmax = 0.0;
    for (int l = 0; l < 2; ++l) {
        const double p = tb_admm_flow(base, prm, 2 * l), q = tb_admm_flow(base, prm, 2 * l + 1);
        h[l] = (p * p + q * q) + x[4 + l];
        const double a = tb_admm_absd(h[l]);
        if (!(a <= hmax)) hmax = a; /* NaN propagates */
    }
    return hmax;
}

/* One augmented-Lagrangian round of one branch after its TRON solve (see
 * tb_admm_options): updates mu / xi in the branch's parameter row and its eta;
 * returns 1 while the branch stays active. */
TB_HD int tb_admm_auglag_update(const double* x, double* prm, double* eta, double feas_tol, double xi_max) {
    double h[2];
    const double hmax = tb_admm_line_hmax(x, prm, h);
    if (hmax <= *eta) {
        if (hmax <= feas_tol) return 0;
        const double xi = prm[TB_BR_XI];
        prm[TB_BR_MU] += xi * h[0];
        prm[TB_BR_MU + 1] += xi * h[1];
        *eta = tb_smax(feas_tol, 0.1 * *eta);
    } else {
        prm[TB_BR_XI] = tb_smin(xi_max, 10.0 * prm[TB_BR_XI]);
    }
    return 1;
}

/* sum_g c2 p^2 + c1 p (generation cost at the component copies) */
TB_HD double tb_admm_gen_cost(const tb_admm_view* v, int g) {
    const double p = v->gen_p[g];
    return v->gen_c2[g] * (p * p) + v->gen_c1[g] * p;
}

#endif /* TB_ADMM_H */
