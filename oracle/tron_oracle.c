/*
 * tron_oracle.c — TEST INFRASTRUCTURE ONLY (see tron_oracle.h).
 *
 * Plain-C restatement of the reference TRON solver.  Each function cites the
 * reference lines it restates (paths relative to /root/reference/proj/).
 * Build flags are part of the contract: -O2 -ffp-contract=off, no -march
 * (SURVEY §8(c)): FMA contraction changes results on nonconvex problems.
 */
#include "tron_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "../paper_2106_14995_b200/csrc/tb_families.h"
#include "../paper_2106_14995_b200/csrc/tb_flops.h"

static __thread long long g_fl; /* per-thread flop counter of the current solve */
static int g_fast_forward = 0; /* opt-in: replay-skip of zero-change fixed points */

void orc_set_fast_forward(int on) { g_fast_forward = on; }

#define SMAX tb_smax /* std::max semantics */
#define SMIN tb_smin /* std::min semantics */

/* ------------------------------------------------------------ dense.hpp */

/* dense.hpp:73-77  y <- y + alpha*x */
void orc_axpy(int n, double alpha, const double* x, double* y) {
    for (int i = 0; i < n; ++i) y[i] += alpha * x[i];
    g_fl += 2 * n;
}

/* dense.hpp:79-84  sequential ascending sum */
double orc_dot(int n, const double* x, const double* y) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += x[i] * y[i];
    g_fl += 2 * n;
    return s;
}

/* dense.hpp:86-88 */
double orc_nrm2(int n, const double* x) {
    g_fl += 1;
    return sqrt(orc_dot(n, x, x));
}

/* dense.hpp:91-94 */
void orc_scal(int n, double alpha, double* x) {
    for (int i = 0; i < n; ++i) x[i] *= alpha;
    g_fl += n;
}

/* dense.hpp:99-121: column sweep with zero-skip on alpha*x_j */
void orc_gemv(int n, double alpha, const double* A, const double* x, double beta, double* y,
              int transpose) {
    for (int i = 0; i < n; ++i) y[i] *= beta;
    if (alpha == 0.0) return;
    if (!transpose) {
        for (int j = 0; j < n; ++j) {
            const double axj = alpha * x[j];
            if (axj == 0.0) continue;
            for (int i = 0; i < n; ++i) y[i] += axj * A[i + (long)j * n];
            g_fl += 2 * n;
        }
    } else {
        for (int j = 0; j < n; ++j) {
            double s = 0.0;
            for (int i = 0; i < n; ++i) s += A[i + (long)j * n] * x[i];
            y[j] += alpha * s;
        }
        g_fl += 2 * n * n;
    }
}

/* dense.hpp:124-127 */
void orc_ccfs(int n, double* A, double alpha) {
    for (int i = 0; i < n; ++i) A[i + (long)i * n] += alpha;
}

/* dense.hpp:51-55: NaN ignored by std::max */
double orc_max_abs(int n, const double* A) {
    double m = 0.0;
    for (long k = 0; k < (long)n * n; ++k) m = SMAX(m, fabs(A[k]));
    return m;
}

/* dense.hpp:138-156: left-looking, zero-skip on L(j,k), division by d */
int orc_chol_left(int n, const double* A, double shift, double* L) {
    memset(L, 0, sizeof(double) * (size_t)n * n);
    for (int j = 0; j < n; ++j) {
        for (int i = j; i < n; ++i) L[i + (long)j * n] = A[i + (long)j * n];
        L[j + (long)j * n] += shift;
        g_fl += 1;
        for (int k = 0; k < j; ++k) {
            const double ljk = L[j + (long)k * n];
            if (ljk == 0.0) continue;
            for (int i = j; i < n; ++i) L[i + (long)j * n] -= ljk * L[i + (long)k * n];
            g_fl += 2 * (n - j);
        }
        const double pivot = L[j + (long)j * n];
        if (!(pivot > 0.0)) return 0;
        const double d = sqrt(pivot);
        L[j + (long)j * n] = d;
        for (int i = j + 1; i < n; ++i) L[i + (long)j * n] /= d;
        g_fl += 1 + (n - j - 1);
    }
    return 1;
}

/* dense.hpp:160-180: right-looking (cross-check only) */
int orc_chol_right(int n, const double* A, double shift, double* L) {
    memset(L, 0, sizeof(double) * (size_t)n * n);
    for (int j = 0; j < n; ++j) {
        for (int i = j; i < n; ++i) L[i + (long)j * n] += A[i + (long)j * n];
        L[j + (long)j * n] += shift;
    }
    for (int j = 0; j < n; ++j) {
        const double pivot = L[j + (long)j * n];
        if (!(pivot > 0.0)) return 0;
        const double d = sqrt(pivot);
        L[j + (long)j * n] = d;
        for (int i = j + 1; i < n; ++i) L[i + (long)j * n] /= d;
        for (int k = j + 1; k < n; ++k) {
            const double lkj = L[k + (long)j * n];
            if (lkj == 0.0) continue;
            for (int i = k; i < n; ++i) L[i + (long)k * n] -= L[i + (long)j * n] * lkj;
        }
    }
    return 1;
}

/* dense.hpp:182-201 shifted_factorize: alpha = 0, then max(2 alpha, alpha0)
 * up to cap = 1e8 * max(1, max_abs(A)) */
/* diagnostics: histogram of attempts per shifted_factorize call */
static long g_ccf_hist[64];
/* the device's closed form of t shift-escalation steps (tb_math.h), for the
 * CPU test that pins it to the reference's iteration (dense.hpp:197) */
double orc_debug_shift_ahead(double a, double alpha0, int t) { return tb_shift_ahead(a, alpha0, t); }

void orc_debug_ccf_hist(long* out, int clear) {
    for (int k = 0; k < 64; ++k) {
        out[k] = __atomic_load_n(&g_ccf_hist[k], __ATOMIC_RELAXED);
        if (clear) __atomic_store_n(&g_ccf_hist[k], 0, __ATOMIC_RELAXED);
    }
}
/* diagnostics: histogram of free-set sizes nf per face pass (bins of 8) */
static long g_nf_hist[17];
void orc_debug_nf_hist(long* out, int clear) {
    for (int k = 0; k < 17; ++k) {
        out[k] = __atomic_load_n(&g_nf_hist[k], __ATOMIC_RELAXED);
        if (clear) __atomic_store_n(&g_nf_hist[k], 0, __ATOMIC_RELAXED);
    }
}
static void ccf_hist_add(int attempts) {
    __atomic_fetch_add(&g_ccf_hist[attempts < 63 ? attempts : 63], 1, __ATOMIC_RELAXED);
}

static int orc_shifted_factorize(int n, const double* A, double* L, double* shift, int left) {
    double max_diag = 0.0;
    for (int i = 0; i < n; ++i) max_diag = SMAX(max_diag, fabs(A[i + (long)i * n]));
    const double alpha0 = SMAX(1e-3 * max_diag, 1e-8);
    const double cap = 1e8 * SMAX(1.0, orc_max_abs(n, A));
    double alpha = 0.0;
    for (int att = 1;; ++att) {
        const int ok = left ? orc_chol_left(n, A, alpha, L) : orc_chol_right(n, A, alpha, L);
        if (ok) {
            *shift = alpha;
            ccf_hist_add(att);
            return 0;
        }
        alpha = SMAX(2.0 * alpha, alpha0);
        g_fl += 1;
        if (!(alpha <= cap)) {
            ccf_hist_add(0);
            return TB_STATUS_FACTORIZATION_FAILED;
        }
    }
}

/* dense.hpp:208-210 */
int orc_ccf(int n, const double* A, double* L, double* shift) {
    return orc_shifted_factorize(n, A, L, shift, 1);
}
/* dense.hpp:213-215 */
int orc_ccf_right(int n, const double* A, double* L, double* shift) {
    return orc_shifted_factorize(n, A, L, shift, 0);
}

/* dense.hpp:218-237: upfront zero-diagonal check, forward row dot-form,
 * backward ascending-j dot-form */
int orc_trtrs(int n, const double* L, double* b, int transpose) {
    for (int i = 0; i < n; ++i)
        if (L[i + (long)i * n] == 0.0) return TB_STATUS_SINGULAR_FACTOR;
    if (!transpose) {
        for (int i = 0; i < n; ++i) {
            double s = b[i];
            for (int j = 0; j < i; ++j) s -= L[i + (long)j * n] * b[j];
            b[i] = s / L[i + (long)i * n];
        }
    } else {
        for (int i = n - 1; i >= 0; --i) {
            double s = b[i];
            for (int j = i + 1; j < n; ++j) s -= L[j + (long)i * n] * b[j];
            b[i] = s / L[i + (long)i * n];
        }
    }
    g_fl += (long long)n * n;
    return 0;
}

/* ------------------------------------------------------------- tron.hpp */

/* tron.hpp:105-108 */
void orc_clip(int n, double* x, const double* l, const double* u) {
    for (int i = 0; i < n; ++i) x[i] = SMIN(SMAX(x[i], l[i]), u[i]);
}

/* tron.hpp:112-121 */
double orc_pgnorm(int n, const double* x, const double* g, const double* l, const double* u) {
    double norm = 0.0;
    for (int i = 0; i < n; ++i) {
        double pg = g[i];
        if (x[i] <= l[i]) pg = SMIN(g[i], 0.0);
        else if (x[i] >= u[i]) pg = SMAX(g[i], 0.0);
        norm = SMAX(norm, fabs(pg));
    }
    return norm;
}

/* tron.hpp:129-138 */
void orc_gpstep(int n, const double* x, double alpha, const double* w, const double* l,
                const double* u, double* s) {
    for (int i = 0; i < n; ++i) {
        const double trial = x[i] + alpha * w[i];
        if (trial < l[i]) s[i] = l[i] - x[i];
        else if (trial > u[i]) s[i] = u[i] - x[i];
        else s[i] = alpha * w[i];
    }
    g_fl += 2 * n;
}

/* tron.hpp:147-164 */
void orc_breakpt(int n, const double* x, const double* w, const double* l, const double* u,
                 int* count, double* bmin, double* bmax) {
    int c = 0;
    double mn = 0.0, mx = 0.0;
    for (int i = 0; i < n; ++i) {
        double b;
        if (x[i] < u[i] && w[i] > 0.0) b = (u[i] - x[i]) / w[i];
        else if (x[i] > l[i] && w[i] < 0.0) b = (l[i] - x[i]) / w[i];
        else continue;
        if (!isfinite(b)) continue;
        if (c == 0) {
            mn = mx = b;
        } else {
            mn = SMIN(mn, b);
            mx = SMAX(mx, b);
        }
        ++c;
    }
    g_fl += 2 * n;
    *count = c;
    *bmin = mn;
    *bmax = mx;
}

/* tron.hpp:167-176 */
int orc_trqsol(int n, const double* x, const double* w, double delta, double* sigma) {
    const double ptx = orc_dot(n, w, x);
    const double ptp = orc_dot(n, w, w);
    if (ptp == 0.0) return TB_STATUS_ZERO_DIRECTION;
    const double xtx = orc_dot(n, x, x);
    const double dsq = delta * delta;
    const double rad = sqrt(SMAX(ptx * ptx + ptp * SMAX(dsq - xtx, 0.0), 0.0));
    g_fl += 8;
    if (ptx > 0.0) *sigma = (dsq - xtx) / (ptx + rad);
    else *sigma = (rad - ptx) / ptp;
    return 0;
}

/* tron.hpp:185-188 */
double orc_quad_model(int n, const double* A, const double* g, const double* s) {
    double as[n > 0 ? n : 1];
    for (int i = 0; i < n; ++i) as[i] = 0.0;
    orc_gemv(n, 1.0, A, s, 0.0, as, 0);
    g_fl += 2;
    return orc_dot(n, g, s) + 0.5 * orc_dot(n, s, as);
}

/* tron.hpp:201-250 (checked_quad_model :190-194 throws EvaluationError) */
int orc_cauchy(int n, const double* x, const double* g, const double* A, const double* l,
               const double* u, double delta, const tb_tron_config* cfg, double alpha_start,
               double* alpha_out, double* s) {
    const double radius = cfg->mu1 * delta;
    const double extrap_factor = 1.0 / cfg->interp_factor;
    double alpha = alpha_start;
    double minus_g[n > 0 ? n : 1];
    for (int i = 0; i < n; ++i) minus_g[i] = -1.0 * g[i];
    g_fl += n;
    int bcount;
    double bmin, bmax;
    orc_breakpt(n, x, minus_g, l, u, &bcount, &bmin, &bmax);

    orc_gpstep(n, x, -alpha, g, l, u, s);
    int interpolate;
    if (orc_nrm2(n, s) > radius) {
        interpolate = 1;
    } else {
        const double q = orc_quad_model(n, A, g, s);
        if (!isfinite(q)) return TB_STATUS_EVALUATION_ERROR;
        g_fl += 1;
        interpolate = q >= cfg->mu0 * orc_dot(n, g, s);
    }

    if (interpolate) {
        int search = 1;
        while (search && alpha > 1e-30) {
            alpha *= cfg->interp_factor;
            orc_gpstep(n, x, -alpha, g, l, u, s);
            if (orc_nrm2(n, s) <= radius) {
                const double q = orc_quad_model(n, A, g, s);
                if (!isfinite(q)) return TB_STATUS_EVALUATION_ERROR;
                g_fl += 1;
                search = q >= cfg->mu0 * orc_dot(n, g, s);
            }
        }
    } else {
        double alpha_good = alpha;
        int search = 1;
        while (search && alpha <= bmax) {
            alpha *= extrap_factor;
            orc_gpstep(n, x, -alpha, g, l, u, s);
            if (orc_nrm2(n, s) <= radius) {
                const double q = orc_quad_model(n, A, g, s);
                if (!isfinite(q)) return TB_STATUS_EVALUATION_ERROR;
                g_fl += 1;
                if (q < cfg->mu0 * orc_dot(n, g, s)) alpha_good = alpha;
                else search = 0;
            } else {
                search = 0;
            }
        }
        alpha = alpha_good;
        orc_gpstep(n, x, -alpha, g, l, u, s);
    }
    *alpha_out = alpha;
    return 0;
}

/* tron.hpp:259-264 */
int orc_select_free_set(int n, const double* x, const double* l, const double* u, int* free_set) {
    int nf = 0;
    for (int i = 0; i < n; ++i)
        if (l[i] < x[i] && x[i] < u[i]) free_set[nf++] = i;
    return nf;
}

/* tron.hpp:290-344 Steihaug PCG in preconditioned coordinates */
int orc_precond_cg(int n, const double* A, const double* g, const double* L, double delta,
                   const tb_tron_config* cfg, double* step, int* cg_status, int* iterations,
                   double* rel_residual) {
    const int m = n > 0 ? n : 1;
    double w[m], bhat[m], r[m], p[m], z[m], q[m];
    int rc;
    for (int i = 0; i < n; ++i) w[i] = 0.0;
    for (int i = 0; i < n; ++i) bhat[i] = g[i] * -1.0;
    g_fl += n;
    if ((rc = orc_trtrs(n, L, bhat, 0))) return rc;
    const double bnorm = orc_nrm2(n, bhat);
    *iterations = 0;
    *rel_residual = 0.0;
    if (bnorm == 0.0) {
        for (int i = 0; i < n; ++i) step[i] = 0.0;
        *cg_status = 0;
        return 0;
    }
    memcpy(r, bhat, sizeof(double) * n);
    memcpy(p, r, sizeof(double) * n);
    double rho = orc_dot(n, r, r);
    *cg_status = 3; /* IterCap */
    for (int k = 1; k <= n; ++k) {
        *iterations = k;
        memcpy(z, p, sizeof(double) * n);
        if ((rc = orc_trtrs(n, L, z, 1))) return rc;
        for (int i = 0; i < n; ++i) q[i] = 0.0;
        orc_gemv(n, 1.0, A, z, 0.0, q, 0);
        if ((rc = orc_trtrs(n, L, q, 0))) return rc;
        const double ptq = orc_dot(n, p, q);
        if (ptq <= 0.0) {
            double sigma;
            if ((rc = orc_trqsol(n, w, p, delta, &sigma))) return rc;
            orc_axpy(n, sigma, p, w);
            *cg_status = 2; /* NegCurve */
            break;
        }
        const double alpha = rho / ptq;
        double sigma;
        if ((rc = orc_trqsol(n, w, p, delta, &sigma))) return rc;
        g_fl += 1;
        if (alpha >= sigma) {
            orc_axpy(n, sigma, p, w);
            *cg_status = 1; /* Boundary */
            break;
        }
        orc_axpy(n, alpha, p, w);
        orc_axpy(n, -alpha, q, r);
        const double rtr = orc_dot(n, r, r);
        g_fl += 2;
        if (sqrt(rtr) <= cfg->cg_tol * bnorm) {
            *cg_status = 0;
            break;
        }
        orc_scal(n, rtr / rho, p); /* p = axpy(1.0, r, scal(rtr/rho, p)) (:335) */
        orc_axpy(n, 1.0, r, p);
        g_fl += 1;
        rho = rtr;
    }
    /* :340-341 diagnostic; not counted (never read by solve) */
    {
        const long long fl_save = g_fl;
        double t[m], aw[m];
        memcpy(t, w, sizeof(double) * n);
        if ((rc = orc_trtrs(n, L, t, 1))) return rc;
        for (int i = 0; i < n; ++i) aw[i] = 0.0;
        orc_gemv(n, 1.0, A, t, 0.0, aw, 0);
        if ((rc = orc_trtrs(n, L, aw, 0))) return rc;
        double res[m];
        memcpy(res, bhat, sizeof(double) * n);
        orc_axpy(n, -1.0, aw, res);
        *rel_residual = orc_nrm2(n, res) / bnorm;
        g_fl = fl_save;
    }
    memcpy(step, w, sizeof(double) * n);
    return orc_trtrs(n, L, step, 1);
}

/* tron.hpp:354-374 */
void orc_line_search(int n, const double* x, const double* l, const double* u, const double* A,
                     const double* g, const double* w, const tb_tron_config* cfg, double* beta_out,
                     double* x_next) {
    const double kBetaFloor = 1e-12;
    const int m = n > 0 ? n : 1;
    double beta = 1.0;
    int bcount;
    double bmin, bmax;
    orc_breakpt(n, x, w, l, u, &bcount, &bmin, &bmax);
    int search = 1;
    double s[m];
    while (search && beta > bmin && beta > kBetaFloor) {
        orc_gpstep(n, x, beta, w, l, u, s);
        const double q = orc_quad_model(n, A, g, s);
        g_fl += 1;
        if (q <= cfg->mu0 * orc_dot(n, g, s)) search = 0;
        else beta *= cfg->interp_factor;
    }
    if (beta < 1.0 && beta < bmin) beta = bmin;
    memcpy(x_next, x, sizeof(double) * n);
    orc_axpy(n, beta, w, x_next);
    orc_clip(n, x_next, l, u);
    *beta_out = beta;
}

/* tron.hpp:394-447 detail::subspace_step */
static int orc_subspace_step(int n, const double* x0, const double* g, const double* A,
                             const double* l, const double* u, double delta,
                             const tb_tron_config* cfg, const double* cauchy_s, double* x_out,
                             double* step, long long* cg_iterations) {
    const int m = n > 0 ? n : 1;
    int rc;
    memcpy(x_out, x0, sizeof(double) * n);
    orc_axpy(n, 1.0, cauchy_s, x_out);
    orc_clip(n, x_out, l, u);
    double* s = step;
    for (int i = 0; i < n; ++i) s[i] = x_out[i] - x0[i];
    g_fl += n;
    double w[m];
    for (int i = 0; i < n; ++i) w[i] = 0.0;
    orc_gemv(n, 1.0, A, s, 0.0, w, 0);
    *cg_iterations = 0;

    int F[m];
    double* B = (double*)malloc(sizeof(double) * (size_t)m * m);
    double* Lf = (double*)malloc(sizeof(double) * (size_t)m * m);
    for (int faces = 0; faces < n; ++faces) {
        const int nf = orc_select_free_set(n, x_out, l, u, F);
        __atomic_fetch_add(&g_nf_hist[(nf + 7) / 8 < 16 ? (nf + 7) / 8 : 16], 1, __ATOMIC_RELAXED);
        if (nf == 0) break;
        for (int j = 0; j < nf; ++j)
            for (int i = 0; i < nf; ++i) B[i + (long)j * nf] = A[F[i] + (long)F[j] * n];
        double shift;
        if ((rc = orc_ccf(nf, B, Lf, &shift))) goto out;
        double gfree[m], gorig[m];
        for (int j = 0; j < nf; ++j) {
            gfree[j] = w[F[j]] + g[F[j]];
            gorig[j] = g[F[j]];
        }
        g_fl += nf;
        const double gfnorm = orc_nrm2(nf, gorig);
        double cstep[m];
        int cg_status, cg_its;
        double relres;
        if ((rc = orc_precond_cg(nf, B, gfree, Lf, delta, cfg, cstep, &cg_status, &cg_its, &relres)))
            goto out;
        *cg_iterations += cg_its;
        double xf[m], lf[m], uf[m], xn[m];
        for (int j = 0; j < nf; ++j) {
            xf[j] = x_out[F[j]];
            lf[j] = l[F[j]];
            uf[j] = u[F[j]];
        }
        double beta;
        orc_line_search(nf, xf, lf, uf, B, gfree, cstep, cfg, &beta, xn);
        for (int j = 0; j < nf; ++j) {
            x_out[F[j]] = xn[j];
            s[F[j]] += xn[j] - xf[j];
        }
        g_fl += 2 * nf;
        for (int i = 0; i < n; ++i) w[i] = 0.0;
        orc_gemv(n, 1.0, A, s, 0.0, w, 0);
        double gfnormf = 0.0;
        for (int j = 0; j < nf; ++j) {
            const double t = w[F[j]] + g[F[j]];
            gfnormf += t * t;
        }
        g_fl += 3 * nf + 2;
        if (sqrt(gfnormf) <= cfg->cg_tol * gfnorm) break;
        if (cg_status == 1 || cg_status == 3) break;
    }
    rc = 0;
out:
    free(B);
    free(Lf);
    return rc;
}

/* tron.hpp:453-549 solve */
int orc_solve(const orc_problem* p, const double* x0, const tb_tron_config* cfg, double* x_star,
              orc_report* rep) {
    const int n = p->n;
    const int m = n > 0 ? n : 1;
    const double* l = p->lower;
    const double* u = p->upper;
    const double kEta1 = 0.25, kEta2 = 0.75;
    int rc = 0;
    g_fl = 0;
    memset(rep, 0, sizeof(*rep));
    rep->status = TB_STATUS_ITER_LIMIT;
    for (int i = 0; i < n; ++i)
        if (!(l[i] <= u[i])) {
            rep->status = TB_STATUS_INVALID_BOUNDS;
            return TB_STATUS_INVALID_BOUNDS;
        }

    double* x = x_star;
    memcpy(x, x0, sizeof(double) * n);
    orc_clip(n, x, l, u);
    double f = p->f(p->ctx, x);
    rep->f_evals = 1;
    double g[m], xs[m], s[m], As[m];
    p->grad(p->ctx, x, g);
    double pg = orc_pgnorm(n, x, g, l, u);
    double delta = cfg->has_delta0 ? cfg->delta0 : SMAX(orc_nrm2(n, g), 1.0);
    double alpha_c = 1.0;
    double* A = (double*)malloc(sizeof(double) * (size_t)m * m);
    int need_hessian = 1;
    rep->status = pg <= cfg->tol_pg ? TB_STATUS_CONVERGED : TB_STATUS_ITER_LIMIT;

    if (rep->status != TB_STATUS_CONVERGED) {
        for (int iter = 1; iter <= cfg->max_iter; ++iter) {
            rep->iterations = iter;
            ++rep->executed_iterations;
            if (need_hessian) {
                p->hess(p->ctx, x, A);
                need_hessian = 0;
            }
            const long long fl_iter0 = g_fl;
            const double delta_in = delta, alpha_in = alpha_c;
            double cs[m];
            double alpha_new;
            if ((rc = orc_cauchy(n, x, g, A, l, u, delta, cfg, alpha_c, &alpha_new, cs))) {
                rep->status = rc;
                break;
            }
            alpha_c = alpha_new;
            long long cg_its = 0;
            rc = orc_subspace_step(n, x, g, A, l, u, delta, cfg, cs, xs, s, &cg_its);
            if (rc == TB_STATUS_FACTORIZATION_FAILED) {
                rep->status = TB_STATUS_FACTORIZATION_FAILED;
                rc = 0;
                break;
            }
            if (rc) {
                rep->status = rc;
                break;
            }
            rep->cg_iterations += cg_its;
            const double f_trial = p->f(p->ctx, xs);
            ++rep->f_evals;

            const double gs = orc_dot(n, g, s);
            for (int i = 0; i < n; ++i) As[i] = 0.0;
            orc_gemv(n, 1.0, A, s, 0.0, As, 0);
            const double prered = -(gs + 0.5 * orc_dot(n, s, As));
            const double actred = f - f_trial;
            const double snorm = orc_nrm2(n, s);
            g_fl += 4;
            if (iter == 1) delta = SMIN(delta, snorm);

            double alphax;
            if (f_trial - f - gs <= 0.0) alphax = cfg->sigma3;
            else alphax = SMAX(cfg->sigma1, -0.5 * (gs / (f_trial - f - gs)));

            if (actred < cfg->eta0 * prered)
                delta = SMIN(SMAX(alphax, cfg->sigma1) * snorm, cfg->sigma2 * delta);
            else if (actred < kEta1 * prered)
                delta = SMAX(cfg->sigma1 * delta, SMIN(alphax * snorm, cfg->sigma2 * delta));
            else if (actred < kEta2 * prered)
                delta = SMAX(cfg->sigma1 * delta, SMIN(alphax * snorm, cfg->sigma3 * delta));
            else
                delta = SMAX(delta, SMIN(alphax * snorm, cfg->sigma3 * delta));
            delta = SMIN(delta, cfg->delta_max);
            g_fl += 12;

            const int accepted = actred > cfg->eta0 * prered;
            if (accepted) {
                memcpy(x, xs, sizeof(double) * n);
                f = f_trial;
                p->grad(p->ctx, x, g);
                need_hessian = 1;
                pg = orc_pgnorm(n, x, g, l, u);
                if (pg <= cfg->tol_pg) {
                    rep->status = TB_STATUS_CONVERGED;
                    break;
                }
            }
            if (delta <= 1e-300) break;
            /* a rejected iteration k >= 2 leaving delta and
             * alpha_c unchanged leaves the whole state unchanged; the rest of
             * the loop replays it (same counters each time). */
            if (!accepted && iter >= 2 && delta == delta_in && alpha_c == alpha_in) {
                if (!rep->ff_iter) rep->ff_iter = iter;
                if (g_fast_forward) {
                    const long long rem = cfg->max_iter - iter;
                    rep->cg_iterations += rem * cg_its;
                    rep->f_evals += rem;
                    g_fl += rem * (g_fl - fl_iter0);
                    rep->iterations = cfg->max_iter;
                    break;
                }
            }
        }
    }
    free(A);
    rep->f_star = f;
    rep->pg_norm = pg;
    rep->flops = g_fl;
    return rc;
}

/* ------------------------------------------------------- family twins */

typedef struct {
    int fam, n;
    const double* prm;
    long long* fl;
} fam_ctx;

static double fam_f(void* c, const double* x) {
    fam_ctx* fc = (fam_ctx*)c;
    g_fl += tb_family_flops(fc->fam, fc->n, 0);
    return tb_family_f(fc->fam, x, fc->prm, fc->n);
}
static void fam_g(void* c, const double* x, double* g) {
    fam_ctx* fc = (fam_ctx*)c;
    g_fl += tb_family_flops(fc->fam, fc->n, 1);
    tb_family_grad(fc->fam, x, fc->prm, fc->n, g);
}
static void fam_h(void* c, const double* x, double* A) {
    fam_ctx* fc = (fam_ctx*)c;
    g_fl += tb_family_flops(fc->fam, fc->n, 2);
    tb_family_hess(fc->fam, x, fc->prm, fc->n, A);
}

int orc_solve_family(int family, int n, const double* x0, const double* l, const double* u,
                     const double* params, const tb_tron_config* cfg, double* x_star,
                     orc_report* rep) {
    fam_ctx fc = {family, n, params, 0};
    orc_problem p = {n, l, u, fam_f, fam_g, fam_h, &fc};
    return orc_solve(&p, x0, cfg, x_star, rep);
}

void orc_family_eval(int family, int n, const double* x, const double* params, double* f,
                     double* g, double* H) {
    if (f) *f = tb_family_f(family, x, params, n);
    if (g) tb_family_grad(family, x, params, n, g);
    if (H) tb_family_hess(family, x, params, n, H);
}

/* ---------------------------------------------------------- batch.hpp */

typedef struct {
    int family, n;
    int64_t lo, hi;
    const double *x0, *lower, *upper, *params;
    int64_t stride;
    const tb_tron_config* cfg;
    double *x_star, *f_star, *pg_norm;
    int32_t *status, *iterations;
    int64_t *cg_iterations, *f_evals, *flops;
    int32_t *executed, *ff_iter;
    int err;
} chunk_t;

static void* run_chunk(void* arg) {
    chunk_t* c = (chunk_t*)arg;
    c->err = 0;
    for (int64_t i = c->lo; i < c->hi; ++i) {
        const int n = c->n;
        orc_report rep;
        const double* prm = c->params ? c->params + i * c->stride : NULL;
        const int rc = orc_solve_family(c->family, n, c->x0 + i * n, c->lower + i * n,
                                        c->upper + i * n, prm, c->cfg, c->x_star + i * n, &rep);
        if (c->f_star) c->f_star[i] = rep.f_star;
        if (c->pg_norm) c->pg_norm[i] = rep.pg_norm;
        if (c->status) c->status[i] = rep.status;
        if (c->iterations) c->iterations[i] = rep.iterations;
        if (c->cg_iterations) c->cg_iterations[i] = rep.cg_iterations;
        if (c->f_evals) c->f_evals[i] = rep.f_evals;
        if (c->flops) c->flops[i] = rep.flops;
        if (c->executed) c->executed[i] = rep.executed_iterations;
        if (c->ff_iter) c->ff_iter[i] = rep.ff_iter;
        if (rc && !c->err) c->err = rc; /* reference aborts the chunk; we record */
    }
    return NULL;
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

int orc_solve_batch(int family, int n, int64_t count, const double* x0, const double* lower,
                    const double* upper, const double* params, int64_t params_stride,
                    const tb_tron_config* cfg, int workers, double* x_star, double* f_star,
                    double* pg_norm, int32_t* status, int32_t* iterations, int64_t* cg_iterations,
                    int64_t* f_evals, int64_t* flops, int32_t* executed, int32_t* ff_iter,
                    double* batch_wall_time) {
    if (workers < 1) return TB_E_INVALID_ARGUMENT;
    chunk_t* ch = (chunk_t*)calloc((size_t)workers, sizeof(chunk_t));
    pthread_t* th = (pthread_t*)calloc((size_t)workers, sizeof(pthread_t));
    const int64_t base = count / workers, rem = count % workers;
    int64_t lo = 0;
    const double t0 = now_s();
    for (int k = 0; k < workers; ++k) {
        const int64_t hi = lo + base + (k < rem ? 1 : 0);
        chunk_t c = {family, n, lo, hi, x0, lower, upper, params, params_stride, cfg,
                     x_star, f_star, pg_norm, status, iterations, cg_iterations, f_evals, flops,
                     executed, ff_iter, 0};
        ch[k] = c;
        lo = hi;
    }
    if (workers == 1) {
        run_chunk(&ch[0]);
    } else {
        for (int k = 0; k < workers; ++k) pthread_create(&th[k], NULL, run_chunk, &ch[k]);
        for (int k = 0; k < workers; ++k) pthread_join(th[k], NULL);
    }
    if (batch_wall_time) *batch_wall_time = now_s() - t0;
    int err = 0;
    for (int k = 0; k < workers && !err; ++k) err = ch[k].err;
    free(ch);
    free(th);
    return err;
}

/* batch.hpp:89-111 */
int orc_imbalance(const double* times, int n_iters, int n_parts, double* nu, double* nu_max,
                  double* nu_min, double* nu_mean) {
    if (n_iters < 1 || n_parts < 2) return TB_E_INVALID_ARGUMENT;
    for (int k = 0; k < n_iters; ++k) {
        double tmax = 0.0, tsum = 0.0;
        for (int p = 0; p < n_parts; ++p) {
            const double t = times[(long)k * n_parts + p];
            if (!(t > 0.0)) return TB_E_INVALID_ARGUMENT;
            tmax = SMAX(tmax, t);
            tsum += t;
        }
        const double tmean = tsum / (double)n_parts;
        nu[k] = (tmax / tmean - 1.0) * 100.0;
    }
    double mx = nu[0], mn = nu[0], s = 0.0;
    for (int k = 0; k < n_iters; ++k) {
        if (mx < nu[k]) mx = nu[k];
        if (nu[k] < mn) mn = nu[k];
        s += nu[k];
    }
    *nu_max = mx;
    *nu_min = mn;
    *nu_mean = s / (double)n_iters;
    return 0;
}

/* tron.hpp:54-68 */
void orc_config_default(tb_tron_config* c) {
    memset(c, 0, sizeof(*c));
    c->tol_pg = 1e-6;
    c->has_delta0 = 0;
    c->delta0 = 0.0;
    c->max_iter = 200;
    c->cg_tol = 0.1;
    c->eta0 = 1e-4;
    c->sigma1 = 0.25;
    c->sigma2 = 0.5;
    c->sigma3 = 4.0;
    c->mu0 = 1e-2;
    c->mu1 = 1.0;
    c->interp_factor = 0.5;
    c->delta_max = 1e10;
}

/* tron.hpp:70-80 */
int orc_config_validate(const tb_tron_config* c, const char** msg) {
    if (!(c->tol_pg > 0.0)) { *msg = "TronConfig: tol_pg must be > 0"; return 1; }
    if (c->has_delta0 && !(c->delta0 > 0.0)) { *msg = "TronConfig: delta0 must be > 0"; return 1; }
    if (!(0.0 < c->sigma1 && c->sigma1 < c->sigma2 && c->sigma2 < 1.0 && 1.0 < c->sigma3)) {
        *msg = "TronConfig: need 0 < sigma1 < sigma2 < 1 < sigma3";
        return 1;
    }
    if (!(0.0 < c->eta0 && c->eta0 < 1.0)) { *msg = "TronConfig: need 0 < eta0 < 1"; return 1; }
    if (!(0.0 < c->mu0 && c->mu0 < 1.0)) { *msg = "TronConfig: need 0 < mu0 < 1"; return 1; }
    if (!(0.0 < c->interp_factor && c->interp_factor < 1.0)) {
        *msg = "TronConfig: need 0 < interp_factor < 1";
        return 1;
    }
    if (c->max_iter < 1) { *msg = "TronConfig: max_iter must be >= 1"; return 1; }
    *msg = "";
    return 0;
}
