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
/* Per-evaluation shared subexpressions of Eq. (3): flows, their gradients
 * w.r.t. z = (v_i, v_j, th_i, th_j), and the multiplier-like coefficients
 * lambda + rho * residual.  Flows:
 *   p_ij =  gff w_i + gft wR + bft wI      q_ij = -bff w_i - bft wR + gft wI
 *   p_ji =  gtt w_j + gtf wR - btf wI      q_ji = -btt w_j - btf wR - gtf wI
 * with w_i = v_i^2, wR = v_i v_j cos(th_i - th_j), wI = v_i v_j sin(...). */
typedef struct {
    int n;
    double vi, vj, cs, sn, wR, wI, wi, wj;
    double fa[4], fb[4], fc[4]; /* F = fa*w_own + fb*wR + fc*wI */
    double F[4];
    double dF[4][4];
    double cF[4];              /* lam + rho * (F - F~) */
    double rw[2], cw[2];       /* w residual, lam_w + rho_w * rw */
    double rt[2], ct[2];       /* theta residual, lam_t + rho_t * rt */
    double h[2], ch[2];        /* line limit: h = p^2 + q^2 + s, mu + xi h */
    double dh[2][4];
} tb_branch_ctx;

TB_HD void tb_branch_ctx_init(const double* x, const double* prm, int n, tb_branch_ctx* c) {
    c->n = n;
    const double vi = x[0], vj = x[1];
    double sn, cs;
    tb_sincos(x[2] - x[3], &sn, &cs);
    const double vv = vi * vj;
    c->vi = vi; c->vj = vj; c->cs = cs; c->sn = sn;
    c->wR = vv * cs;
    c->wI = vv * sn;
    c->wi = vi * vi;
    c->wj = vj * vj;
    const double gff = prm[TB_BR_GFF], bff = prm[TB_BR_BFF], gft = prm[TB_BR_GFT], bft = prm[TB_BR_BFT];
    const double gtt = prm[TB_BR_GTT], btt = prm[TB_BR_BTT], gtf = prm[TB_BR_GTF], btf = prm[TB_BR_BTF];
    c->fa[0] = gff;  c->fb[0] = gft;  c->fc[0] = bft;
    c->fa[1] = -bff; c->fb[1] = -bft; c->fc[1] = gft;
    c->fa[2] = gtt;  c->fb[2] = gtf;  c->fc[2] = -btf;
    c->fa[3] = -btt; c->fb[3] = -btf; c->fc[3] = -gtf;
    const double dwR[4] = {vj * cs, vi * cs, -c->wI, c->wI};
    const double dwI[4] = {vj * sn, vi * sn, c->wR, -c->wR};
    const double dwi[4] = {2.0 * vi, 0.0, 0.0, 0.0};
    const double dwj[4] = {0.0, 2.0 * vj, 0.0, 0.0};
    for (int f = 0; f < 4; ++f) {
        const double own = f < 2 ? c->wi : c->wj;
        const double* down = f < 2 ? dwi : dwj;
        c->F[f] = (c->fa[f] * own + c->fb[f] * c->wR) + c->fc[f] * c->wI;
        for (int k = 0; k < 4; ++k)
            c->dF[f][k] = (c->fa[f] * down[k] + c->fb[f] * dwR[k]) + c->fc[f] * dwI[k];
        const double r = c->F[f] - prm[TB_BR_TIL + f];
        c->cF[f] = prm[TB_BR_LAM + f] + prm[TB_BR_RHO + f] * r;
    }
    for (int l = 0; l < 2; ++l) {
        const double v = l == 0 ? vi : vj;
        c->rw[l] = v * v - prm[TB_BR_WTIL + l];
        c->cw[l] = prm[TB_BR_LAMW + l] + prm[TB_BR_RHOW + l] * c->rw[l];
        c->rt[l] = x[2 + l] - prm[TB_BR_TTIL + l];
        c->ct[l] = prm[TB_BR_LAMT + l] + prm[TB_BR_RHOT + l] * c->rt[l];
    }
    for (int l = 0; l < 2; ++l) {
        c->h[l] = 0.0; c->ch[l] = 0.0;
        for (int k = 0; k < 4; ++k) c->dh[l][k] = 0.0;
    }
    if (n == 6) {
        for (int l = 0; l < 2; ++l) {
            const double p = c->F[2 * l], q = c->F[2 * l + 1];
            c->h[l] = (p * p + q * q) + x[4 + l];
            c->ch[l] = prm[TB_BR_MU + l] + prm[TB_BR_XI] * c->h[l];
            for (int k = 0; k < 4; ++k)
                c->dh[l][k] = (2.0 * p) * c->dF[2 * l][k] + (2.0 * q) * c->dF[2 * l + 1][k];
        }
    }
}

/* second derivatives of wR / wI, canonical a <= b < 4 */
TB_HD double tb_branch_d2wR(const tb_branch_ctx* c, int a, int b) {
    switch (a * 4 + b) {
        case 1: return c->cs;               /* (vi, vj) */
        case 2: return -(c->vj * c->sn);    /* (vi, th_i) */
        case 3: return c->vj * c->sn;       /* (vi, th_j) */
        case 6: return -(c->vi * c->sn);    /* (vj, th_i) */
        case 7: return c->vi * c->sn;       /* (vj, th_j) */
        case 10: return -c->wR;             /* (th_i, th_i) */
        case 11: return c->wR;              /* (th_i, th_j) */
        case 15: return -c->wR;             /* (th_j, th_j) */
    }
    return 0.0;
}
TB_HD double tb_branch_d2wI(const tb_branch_ctx* c, int a, int b) {
    switch (a * 4 + b) {
        case 1: return c->sn;
        case 2: return c->vj * c->cs;
        case 3: return -(c->vj * c->cs);
        case 6: return c->vi * c->cs;
        case 7: return -(c->vi * c->cs);
        case 10: return -c->wI;
        case 11: return c->wI;
        case 15: return -c->wI;
    }
    return 0.0;
}
TB_HD double tb_branch_d2F(const tb_branch_ctx* c, int f, int a, int b) {
    const int own = f < 2 ? 0 : 1;
    const double d2own = (a == own && b == own) ? 2.0 : 0.0;
    return (c->fa[f] * d2own + c->fb[f] * tb_branch_d2wR(c, a, b)) + c->fc[f] * tb_branch_d2wI(c, a, b);
}

TB_HD double tb_branch_f_ctx(const tb_branch_ctx* c, const double* prm) {
    double f = 0.0;
    for (int k = 0; k < 4; ++k) {
        const double r = c->F[k] - prm[TB_BR_TIL + k];
        f += prm[TB_BR_LAM + k] * r + (0.5 * prm[TB_BR_RHO + k]) * (r * r);
    }
    for (int l = 0; l < 2; ++l)
        f += prm[TB_BR_LAMW + l] * c->rw[l] + (0.5 * prm[TB_BR_RHOW + l]) * (c->rw[l] * c->rw[l]);
    for (int l = 0; l < 2; ++l)
        f += prm[TB_BR_LAMT + l] * c->rt[l] + (0.5 * prm[TB_BR_RHOT + l]) * (c->rt[l] * c->rt[l]);
    if (c->n == 6)
        for (int l = 0; l < 2; ++l)
            f += prm[TB_BR_MU + l] * c->h[l] + (0.5 * prm[TB_BR_XI]) * (c->h[l] * c->h[l]);
    return f;
}

TB_HD double tb_branch_grad_ctx(const tb_branch_ctx* c, int k) {
    if (k >= 4) return c->ch[k - 4];
    double g = 0.0;
    for (int f = 0; f < 4; ++f) g += c->cF[f] * c->dF[f][k];
    if (k < 2) g += c->cw[k] * (2.0 * (k == 0 ? c->vi : c->vj));
    else g += c->ct[k - 2];
    if (c->n == 6) g += c->ch[0] * c->dh[0][k] + c->ch[1] * c->dh[1][k];
    return g;
}

TB_HD double tb_branch_hess_ctx(const tb_branch_ctx* c, const double* prm, int i, int j) {
    const int a = i < j ? i : j;
    const int b = i < j ? j : i;
    double h = 0.0;
    if (b < 4) {
        for (int f = 0; f < 4; ++f)
            h += (prm[TB_BR_RHO + f] * c->dF[f][a]) * c->dF[f][b] + c->cF[f] * tb_branch_d2F(c, f, a, b);
        if (a == b) {
            if (a < 2) {
                const double dv = 2.0 * (a == 0 ? c->vi : c->vj);
                h += (prm[TB_BR_RHOW + a] * dv) * dv + c->cw[a] * 2.0;
            } else {
                h += prm[TB_BR_RHOT + a - 2];
            }
        }
    }
    if (c->n == 6) {
        const double xi = prm[TB_BR_XI];
        for (int l = 0; l < 2; ++l) {
            const double dha = a < 4 ? c->dh[l][a] : (a == 4 + l ? 1.0 : 0.0);
            const double dhb = b < 4 ? c->dh[l][b] : (b == 4 + l ? 1.0 : 0.0);
            double sec = 0.0;
            if (b < 4) {
                const int fp = 2 * l, fq = 2 * l + 1;
                sec = 2.0 * (((c->dF[fp][a] * c->dF[fp][b] + c->F[fp] * tb_branch_d2F(c, fp, a, b)) +
                              c->dF[fq][a] * c->dF[fq][b]) + c->F[fq] * tb_branch_d2F(c, fq, a, b));
            }
            h += (xi * dha) * dhb + c->ch[l] * sec;
        }
    }
    return h;
}

TB_HD double tb_branch_f(const double* x, const double* prm, int n) {
    tb_branch_ctx c;
    tb_branch_ctx_init(x, prm, n, &c);
    return tb_branch_f_ctx(&c, prm);
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
        for (int i = 0; i < n; ++i) g[i] = tb_branch_grad_ctx(&c, i);
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
            for (int i = 0; i < n; ++i) A[i + (long)j * n] = tb_branch_hess_ctx(&c, prm, i, j);
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
