/*
 * tb_families.h — the BoundedProblem families the batched solver evaluates
 * on the device, written once as plain C shared by
 *   - the CUDA kernel (nvcc --fmad=false, sm_100a), and
 *   - the host twins used only by the CPU oracle / reference driver
 *     (gcc/g++ -ffp-contract=off),
 * so both sides evaluate f, grad f and the Hessian with identical bits.
 *
 * The reference's BoundedProblem concept (tron.hpp:28-36) takes arbitrary host
 * callables (FunctionProblem, tron.hpp:39-52).  Host function pointers cannot
 * run on the GPU, so callbacks become compile-time families selected by id.
 * Each family exposes
 *   f(x, prm, n)                      -> objective
 *   grad_i(x, prm, n, i)              -> i-th gradient component
 *   hess_entry(x, prm, n, i, j)       -> Hessian entry (i, j)
 * with per-component evaluation so one warp lane can own one row.
 *
 * Families
 *   HS45   batch.hpp:116-173 (Hs45Problem) — same prefix/suffix products and
 *          the same multiplication order as the reference; params unused.
 *   BOXQP  tests/support/boxqp_oracle.hpp:44-62 (make_quadratic):
 *          f = 0.5 (x-c)' H (x-c) with H*d computed by the reference gemv
 *          (dense.hpp:99-121: column sweep, zero-skip on d_j) and the
 *          sequential dot (dense.hpp:79-84).  params = [H col-major n*n | c n].
 *   NCVX   SURVEY §8(d) synthetic nonconvex family:
 *          f = 0.5 e'He + 0.25 sum k_i e_i^4 + sum a_i sin(x_i), e = x - c,
 *          H symmetric indefinite.  params = [H packed lower col-major
 *          n(n+1)/2 | c n | k n | a n].
 *   BRANCH SPEC.md:336-368 / PAPER.md:564-590 Eq. (3) ADMM branch subproblem
 *          over z = (v_i, v_j, th_i, th_j) (dim 4), plus the line-limit
 *          augmented-Lagrangian variant with slacks (s_ij, s_ji) (dim 6,
 *          SURVEY App. C).  params layout: see TB_BR_* below.
 */
#ifndef TB_FAMILIES_H
#define TB_FAMILIES_H

#include "tb_math.h"

#define TB_FAMILY_HS45 0
#define TB_FAMILY_BOXQP 1
#define TB_FAMILY_NCVX 2
#define TB_FAMILY_BRANCH 3
#define TB_NUM_FAMILIES 4

/* branch parameter layout (36 doubles per branch) */
#define TB_BR_GFF 0 /* Re Y_ff */
#define TB_BR_BFF 1 /* Im Y_ff */
#define TB_BR_GFT 2 /* Re Y_ft */
#define TB_BR_BFT 3 /* Im Y_ft */
#define TB_BR_GTT 4 /* Re Y_tt */
#define TB_BR_BTT 5 /* Im Y_tt */
#define TB_BR_GTF 6 /* Re Y_tf */
#define TB_BR_BTF 7 /* Im Y_tf */
#define TB_BR_LAM 8     /* lambda for (p_ij, q_ij, p_ji, q_ji): 4 */
#define TB_BR_RHO 12    /* rho for the 4 flows */
#define TB_BR_TIL 16    /* consensus (tilde) flows: 4 */
#define TB_BR_LAMW 20   /* lambda_w (i, j) */
#define TB_BR_RHOW 22   /* rho_w (i, j) */
#define TB_BR_WTIL 24   /* w tilde (i, j) */
#define TB_BR_LAMT 26   /* lambda_theta (i, j) */
#define TB_BR_RHOT 28   /* rho_theta (i, j) */
#define TB_BR_TTIL 30   /* theta tilde (i, j) */
#define TB_BR_MU 32     /* line-limit multipliers mu_ij, mu_ji (dim 6) */
#define TB_BR_XI 34     /* line-limit penalty xi (dim 6) */
#define TB_BR_SMAX2 35  /* s-bar^2 (informational; enters via bounds) */
#define TB_BR_NPARAMS 36

TB_HD long tb_fam_nparams(int fam, int n) {
    switch (fam) {
        case TB_FAMILY_HS45: return 0;
        case TB_FAMILY_BOXQP: return (long)n * n + n;
        case TB_FAMILY_NCVX: return (long)n * (n + 1) / 2 + 3L * n;
        case TB_FAMILY_BRANCH: return TB_BR_NPARAMS;
    }
    return -1;
}

/* valid (family, dim) combinations */
TB_HD int tb_family_dim_ok(int fam, int n) {
    if (n < 1) return 0;
    if (fam == TB_FAMILY_BRANCH) return n == 4 || n == 6;
    return fam >= 0 && fam < TB_NUM_FAMILIES;
}

/* ------------------------------------------------------------------ HS45 */
/* batch.hpp:133-137 */
TB_HD double tb_hs45_f(const double* x, int n) {
    double prod = 1.0;
    for (int i = 0; i < n; ++i) prod *= x[i];
    return 120.0 - prod;
}
/* batch.hpp:139-147: g_i = -prefix[i] * suffix[i+1] */
TB_HD double tb_hs45_grad_i(const double* x, int n, int i) {
    double pre = 1.0;
    for (int k = 0; k < i; ++k) pre *= x[k];
    double suf = 1.0;
    for (int k = n - 1; k > i; --k) suf *= x[k];
    return -pre * suf;
}
/* batch.hpp:149-164: h(a,b) = -prefix[a] * mid * suffix[b+1], a < b, mid grown
 * incrementally over x[a+1..b-1]; zero diagonal. */
TB_HD double tb_hs45_hess(const double* x, int n, int i, int j) {
    if (i == j) return 0.0;
    const int a = i < j ? i : j;
    const int b = i < j ? j : i;
    double pre = 1.0;
    for (int k = 0; k < a; ++k) pre *= x[k];
    double suf = 1.0;
    for (int k = n - 1; k > b; --k) suf *= x[k];
    double mid = 1.0;
    for (int k = a + 1; k < b; ++k) mid *= x[k];
    return -pre * mid * suf;
}

/* ----------------------------------------------------------------- BOXQP */
/* (H d)_i with the reference gemv ordering: y_i = 0; for j asc: if d_j != 0:
 * y_i += d_j * H(i,j)   (dense.hpp:104-112 with alpha = 1, beta = 0) */
TB_HD double tb_boxqp_hd_i(const double* x, const double* prm, int n, int i) {
    const double* H = prm;
    const double* c = prm + (long)n * n;
    double y = 0.0 * 0.0;
    for (int j = 0; j < n; ++j) {
        const double dj = 1.0 * (x[j] - c[j]);
        if (dj == 0.0) continue;
        y += dj * H[i + (long)j * n];
    }
    return y;
}
/* boxqp_oracle.hpp:49-53: 0.5 * dot(d, gemv(1, H, d, 0, 0)) */
TB_HD double tb_boxqp_f(const double* x, const double* prm, int n) {
    const double* c = prm + (long)n * n;
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += (x[i] - c[i]) * tb_boxqp_hd_i(x, prm, n, i);
    return 0.5 * s;
}
TB_HD double tb_boxqp_grad_i(const double* x, const double* prm, int n, int i) {
    return tb_boxqp_hd_i(x, prm, n, i);
}
TB_HD double tb_boxqp_hess(const double* prm, int n, int i, int j) {
    return prm[i + (long)j * n];
}

/* ------------------------------------------------------------------ NCVX */
TB_HD long tb_packed_idx(int n, int i, int j) { /* i >= j, lower, col-major */
    return (long)j * n - (long)j * (j - 1) / 2 + (i - j);
}
TB_HD double tb_ncvx_H(const double* prm, int n, int i, int j) {
    return i >= j ? prm[tb_packed_idx(n, i, j)] : prm[tb_packed_idx(n, j, i)];
}
TB_HD double tb_ncvx_he_i(const double* x, const double* prm, int n, int i) {
    const double* c = prm + (long)n * (n + 1) / 2;
    double y = 0.0;
    for (int j = 0; j < n; ++j) y += tb_ncvx_H(prm, n, i, j) * (x[j] - c[j]);
    return y;
}
TB_HD double tb_ncvx_f(const double* x, const double* prm, int n) {
    const double* c = prm + (long)n * (n + 1) / 2;
    const double* k = c + n;
    const double* a = k + n;
    double q = 0.0;
    for (int i = 0; i < n; ++i) q += (x[i] - c[i]) * tb_ncvx_he_i(x, prm, n, i);
    double quart = 0.0;
    for (int i = 0; i < n; ++i) {
        const double e = x[i] - c[i];
        const double e2 = e * e;
        quart += k[i] * (e2 * e2);
    }
    double sn = 0.0;
    for (int i = 0; i < n; ++i) sn += a[i] * tb_sin(x[i]);
    return (0.5 * q + 0.25 * quart) + sn;
}
TB_HD double tb_ncvx_grad_i(const double* x, const double* prm, int n, int i) {
    const double* c = prm + (long)n * (n + 1) / 2;
    const double* k = c + n;
    const double* a = k + n;
    const double e = x[i] - c[i];
    const double e3 = (e * e) * e;
    return (tb_ncvx_he_i(x, prm, n, i) + k[i] * e3) + a[i] * tb_cos(x[i]);
}
TB_HD double tb_ncvx_hess(const double* x, const double* prm, int n, int i, int j) {
    const double h = tb_ncvx_H(prm, n, i, j);
    if (i != j) return h;
    const double* c = prm + (long)n * (n + 1) / 2;
    const double* k = c + n;
    const double* a = k + n;
    const double e = x[i] - c[i];
    return (h + (3.0 * k[i]) * (e * e)) - a[i] * tb_sin(x[i]);
}

/* ---------------------------------------------------------------- BRANCH */
/* Eq. (3) over z = (v_i, v_j, th_i, th_j) [+ slacks (s_ij, s_ji) at dim 6].
 * Flows, w_i = v_i^2,
 * wR = v_i v_j cos(th_i - th_j), wI = v_i v_j sin(th_i - th_j):
 *   p_ij =  gff w_i + gft wR + bft wI      q_ij = -bff w_i - bft wR + gft wI
 *   p_ji =  gtt w_j + gtf wR - btf wI      q_ji = -btt w_j - btf wR - gtf wI
 * Objective: sum_F lam_F r_F + rho_F/2 r_F^2 (r_F = F - F~) over the four
 * flows, + the same for w_l = v_l^2 and th_l (l = i, j); dim 6 adds, per line
 * end, mu h + xi/2 h^2 with h = p^2 + q^2 + s.
 *
 * Everything an evaluation point needs is a "context" of independent pieces
 * (base terms, one block per flow, per voltage coupling, per line end, and
 * the 4x4 second-derivative tables of wR / wI).  Each piece has one function
 * used by both the host twin (sequentially) and the device (one lane per
 * piece, context in shared memory), so both produce identical bits. */
typedef struct {
    double base[8]; /* vi, vj, cs, sn, wR, wI, wi, wj */
    double F[4];
    double dF[4][4];
    double cF[4];   /* lam + rho * (F - F~) */
    double rw[2], cw[2], rt[2], ct[2];
    double h[2], ch[2];
    double dh[2][4];
    double d2wR[16], d2wI[16]; /* symmetric 4x4, [a*4 + b] */
} tb_branch_ctx;

enum { TB_BRB_VI, TB_BRB_VJ, TB_BRB_CS, TB_BRB_SN, TB_BRB_WR, TB_BRB_WI, TB_BRB_WII, TB_BRB_WJJ };

TB_HD void tb_br_base(const double* x, double* b) {
    const double vi = x[0], vj = x[1];
    double sn, cs;
    tb_sincos(x[2] - x[3], &sn, &cs);
    const double vv = vi * vj;
    b[TB_BRB_VI] = vi;
    b[TB_BRB_VJ] = vj;
    b[TB_BRB_CS] = cs;
    b[TB_BRB_SN] = sn;
    b[TB_BRB_WR] = vv * cs;
    b[TB_BRB_WI] = vv * sn;
    b[TB_BRB_WII] = vi * vi;
    b[TB_BRB_WJJ] = vj * vj;
}

/* F = fa * w_own + fb * wR + fc * wI:
 *   f = 0 (p_ij):  gff,  gft,  bft      f = 1 (q_ij): -bff, -bft,  gft
 *   f = 2 (p_ji):  gtt,  gtf, -btf      f = 3 (q_ji): -btt, -btf, -gtf
 * Written without a switch (selects on the flow's end and kind: the device
 * evaluates different flows in different lanes of a warp, where a switch
 * serialises); negation is exact, so the values are those of the table. */
TB_HD void tb_br_coef(int f, const double* prm, double* fa, double* fb, double* fc) {
    const int o = f >= 2 ? 4 : 0; /* gtt / btt / gtf / btf sit 4 slots after gff / bff / gft / bft */
    const int q = f & 1;          /* reactive flow */
    const double g_own = prm[TB_BR_GFF + o], b_own = prm[TB_BR_BFF + o];
    const double g_x = prm[TB_BR_GFT + o], b_x = prm[TB_BR_BFT + o];
    *fa = q ? -b_own : g_own;
    *fb = q ? -b_x : g_x;
    *fc = q ? (o ? -g_x : g_x) : (o ? -b_x : b_x);
}

/* flow f: value, gradient over z, and lam + rho * residual */
TB_HD void tb_br_flow(int f, const double* b, const double* prm, double* F, double* dF, double* cF) {
    double fa, fb, fc;
    tb_br_coef(f, prm, &fa, &fb, &fc);
    const int own = f < 2 ? 0 : 1;
    const double vi = b[TB_BRB_VI], vj = b[TB_BRB_VJ], cs = b[TB_BRB_CS], sn = b[TB_BRB_SN];
    const double wR = b[TB_BRB_WR], wI = b[TB_BRB_WI];
    const double w_own = own == 0 ? b[TB_BRB_WII] : b[TB_BRB_WJJ];
    const double dwR[4] = {vj * cs, vi * cs, -wI, wI};
    const double dwI[4] = {vj * sn, vi * sn, wR, -wR};
    const double dwo[4] = {own == 0 ? 2.0 * vi : 0.0, own == 1 ? 2.0 * vj : 0.0, 0.0, 0.0};
    *F = (fa * w_own + fb * wR) + fc * wI;
    for (int k = 0; k < 4; ++k) dF[k] = (fa * dwo[k] + fb * dwR[k]) + fc * dwI[k];
    *cF = prm[TB_BR_LAM + f] + prm[TB_BR_RHO + f] * (*F - prm[TB_BR_TIL + f]);
}

/* voltage (w = v^2) and angle couplings of bus end l */
TB_HD void tb_br_volt(int l, const double* x, const double* prm, double* rw, double* cw, double* rt,
                      double* ct) {
    const double v = x[l];
    *rw = v * v - prm[TB_BR_WTIL + l];
    *cw = prm[TB_BR_LAMW + l] + prm[TB_BR_RHOW + l] * *rw;
    *rt = x[2 + l] - prm[TB_BR_TTIL + l];
    *ct = prm[TB_BR_LAMT + l] + prm[TB_BR_RHOT + l] * *rt;
}

/* line-limit term of end l (dim 6): h = p^2 + q^2 + s */
TB_HD void tb_br_line(int l, const double* x, const double* prm, double p, double q, const double* dp,
                      const double* dq, double* h, double* ch, double* dh) {
    *h = (p * p + q * q) + x[4 + l];
    *ch = prm[TB_BR_MU + l] + prm[TB_BR_XI] * *h;
    for (int k = 0; k < 4; ++k) dh[k] = (2.0 * p) * dp[k] + (2.0 * q) * dq[k];
}

/* second derivatives of wR and wI at (a, b), a, b < 4 (symmetric) */
/*   (vi, vj):     cs,          sn              (vi, th_i): -(vj sn),   vj cs
 *   (vi, th_j):   vj sn,      -(vj cs)         (vj, th_i): -(vi sn),   vi cs
 *   (vj, th_j):   vi sn,      -(vi cs)         (th_i, th_i), (th_j, th_j): -wR, -wI
 *   (th_i, th_j): wR,          wI              (vi, vi), (vj, vj): 0, 0
 * Selects instead of a switch (the device builds the 16 entries in 16 lanes
 * at once); the same products and exact negations as the table. */
TB_HD void tb_br_d2w(int a, int b, const double* bs, double* r, double* i) {
    const int lo = a < b ? a : b, hi = a < b ? b : a;
    const double vi = bs[TB_BRB_VI], vj = bs[TB_BRB_VJ], cs = bs[TB_BRB_CS], sn = bs[TB_BRB_SN];
    const double wR = bs[TB_BRB_WR], wI = bs[TB_BRB_WI];
    const int vt = lo < 2 && hi >= 2; /* voltage - angle */
    const int tt = lo >= 2;           /* angle - angle */
    const int vv = lo == 0 && hi == 1;
    const double v = lo == 0 ? vj : vi;
    const double ps = v * sn, pc = v * cs;
    const double r0 = vt ? ps : (tt ? wR : (vv ? cs : 0.0));
    const double i0 = vt ? pc : (tt ? wI : (vv ? sn : 0.0));
    const int same_angle = tt && lo == hi;
    *r = ((vt && hi == 2) || same_angle) ? -r0 : r0;
    *i = ((vt && hi == 3) || same_angle) ? -i0 : i0;
}

TB_HD double tb_br_d2F(const tb_branch_ctx* c, const double* prm, int f, int a, int b) {
    double fa, fb, fc;
    tb_br_coef(f, prm, &fa, &fb, &fc);
    const int own = f < 2 ? 0 : 1;
    const double d2own = (a == own && b == own) ? 2.0 : 0.0;
    return (fa * d2own + fb * c->d2wR[a * 4 + b]) + fc * c->d2wI[a * 4 + b];
}

TB_HD double tb_br_f(const tb_branch_ctx* c, const double* prm, int n) {
    double f = 0.0;
    for (int k = 0; k < 4; ++k) {
        const double r = c->F[k] - prm[TB_BR_TIL + k];
        f += prm[TB_BR_LAM + k] * r + (0.5 * prm[TB_BR_RHO + k]) * (r * r);
    }
    for (int l = 0; l < 2; ++l)
        f += prm[TB_BR_LAMW + l] * c->rw[l] + (0.5 * prm[TB_BR_RHOW + l]) * (c->rw[l] * c->rw[l]);
    for (int l = 0; l < 2; ++l)
        f += prm[TB_BR_LAMT + l] * c->rt[l] + (0.5 * prm[TB_BR_RHOT + l]) * (c->rt[l] * c->rt[l]);
    if (n == 6)
        for (int l = 0; l < 2; ++l)
            f += prm[TB_BR_MU + l] * c->h[l] + (0.5 * prm[TB_BR_XI]) * (c->h[l] * c->h[l]);
    return f;
}

TB_HD double tb_br_grad(const tb_branch_ctx* c, int n, int k) {
    if (k >= 4) return c->ch[k - 4];
    double g = 0.0;
    for (int f = 0; f < 4; ++f) g += c->cF[f] * c->dF[f][k];
    if (k < 2) g += c->cw[k] * (2.0 * c->base[k]);
    else g += c->ct[k - 2];
    if (n == 6) g += c->ch[0] * c->dh[0][k] + c->ch[1] * c->dh[1][k];
    return g;
}

TB_HD double tb_br_hess(const tb_branch_ctx* c, const double* prm, int n, int i, int j) {
    const int a = i < j ? i : j;
    const int b = i < j ? j : i;
    double h = 0.0;
    if (b < 4) {
        for (int f = 0; f < 4; ++f)
            h += (prm[TB_BR_RHO + f] * c->dF[f][a]) * c->dF[f][b] + c->cF[f] * tb_br_d2F(c, prm, f, a, b);
        if (a == b) {
            if (a < 2) {
                const double dv = 2.0 * c->base[a];
                h += (prm[TB_BR_RHOW + a] * dv) * dv + c->cw[a] * 2.0;
            } else {
                h += prm[TB_BR_RHOT + a - 2];
            }
        }
    }
    if (n == 6) {
        const double xi = prm[TB_BR_XI];
        for (int l = 0; l < 2; ++l) {
            const double dha = a < 4 ? c->dh[l][a] : (a == 4 + l ? 1.0 : 0.0);
            const double dhb = b < 4 ? c->dh[l][b] : (b == 4 + l ? 1.0 : 0.0);
            double sec = 0.0;
            if (b < 4) {
                const int fp = 2 * l, fq = 2 * l + 1;
                sec = 2.0 * (((c->dF[fp][a] * c->dF[fp][b] + c->F[fp] * tb_br_d2F(c, prm, fp, a, b)) +
                              c->dF[fq][a] * c->dF[fq][b]) + c->F[fq] * tb_br_d2F(c, prm, fq, a, b));
            }
            h += (xi * dha) * dhb + c->ch[l] * sec;
        }
    }
    return h;
}

/* host-order construction of the full context (the device builds the same
 * pieces in parallel lanes) */
TB_HD void tb_branch_ctx_init(const double* x, const double* prm, int n, tb_branch_ctx* c) {
    tb_br_base(x, c->base);
    for (int f = 0; f < 4; ++f) tb_br_flow(f, c->base, prm, &c->F[f], c->dF[f], &c->cF[f]);
    for (int l = 0; l < 2; ++l) tb_br_volt(l, x, prm, &c->rw[l], &c->cw[l], &c->rt[l], &c->ct[l]);
    for (int e = 0; e < 16; ++e) tb_br_d2w(e / 4, e % 4, c->base, &c->d2wR[e], &c->d2wI[e]);
    for (int l = 0; l < 2; ++l) {
        c->h[l] = 0.0;
        c->ch[l] = 0.0;
        for (int k = 0; k < 4; ++k) c->dh[l][k] = 0.0;
        if (n == 6)
            tb_br_line(l, x, prm, c->F[2 * l], c->F[2 * l + 1], c->dF[2 * l], c->dF[2 * l + 1], &c->h[l], &c->ch[l],
                       c->dh[l]);
    }
}

TB_HD double tb_branch_f(const double* x, const double* prm, int n) {
    tb_branch_ctx c;
    tb_branch_ctx_init(x, prm, n, &c);
    return tb_br_f(&c, prm, n);
}

/* ------------------------------------------------------- generic dispatch */
TB_HD double tb_family_f(int fam, const double* x, const double* prm, int n) {
    switch (fam) {
        case TB_FAMILY_HS45: return tb_hs45_f(x, n);
        case TB_FAMILY_BOXQP: return tb_boxqp_f(x, prm, n);
        case TB_FAMILY_NCVX: return tb_ncvx_f(x, prm, n);
        default: return tb_branch_f(x, prm, n);
    }
}

/* full gradient / Hessian (host twins and reference driver use these; the
 * device evaluates one component / row per lane with the same functions) */
TB_HD void tb_family_grad(int fam, const double* x, const double* prm, int n, double* g) {
    if (fam == TB_FAMILY_BRANCH) {
        tb_branch_ctx c;
        tb_branch_ctx_init(x, prm, n, &c);
        for (int i = 0; i < n; ++i) g[i] = tb_br_grad(&c, n, i);
        return;
    }
    for (int i = 0; i < n; ++i) {
        if (fam == TB_FAMILY_HS45) g[i] = tb_hs45_grad_i(x, n, i);
        else if (fam == TB_FAMILY_BOXQP) g[i] = tb_boxqp_grad_i(x, prm, n, i);
        else g[i] = tb_ncvx_grad_i(x, prm, n, i);
    }
}

/* column-major n x n: A[i + j*n] */
TB_HD void tb_family_hess(int fam, const double* x, const double* prm, int n, double* A) {
    if (fam == TB_FAMILY_BRANCH) {
        tb_branch_ctx c;
        tb_branch_ctx_init(x, prm, n, &c);
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) A[i + (long)j * n] = tb_br_hess(&c, prm, n, i, j);
        return;
    }
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
            double v;
            if (fam == TB_FAMILY_HS45) v = tb_hs45_hess(x, n, i, j);
            else if (fam == TB_FAMILY_BOXQP) v = tb_boxqp_hess(prm, n, i, j);
            else v = tb_ncvx_hess(x, prm, n, i, j);
            A[i + (long)j * n] = v;
        }
}

#endif /* TB_FAMILIES_H */
