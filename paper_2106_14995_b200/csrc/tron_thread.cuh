// tron_thread.cuh — one THREAD per problem (branch and ncvx families, n = D <= 8).
//
// The warp kernel (tron_device.cuh) spreads one problem over a warp, which
// maximises throughput on large batches, but every reduction / solve step of a
// lone problem then pays a shuffle or a shared-memory round trip.  The ADMM
// branch stage is bounded by its slowest subproblem (~200 TRON
// iterations of one branch set the iteration time), so there the latency of
// ONE problem matters: this form keeps the whole problem in one thread —
// vectors and the 4x4 / 6x6 Hessian and factor in registers, the branch
// evaluation context in local memory — and runs the reference's sequential
// loops directly (tron.hpp / dense.hpp order: ascending sums, left-looking
// factorization with zero-skip, sequential shift attempts, row dot-form
// solves).  The arithmetic is the warp kernel's, so results are bit-identical
// to it and to the reference (tests/test_admm.py, tests/test_gpu_parity.py).
// No flop counting (the COUNT variant stays in the warp kernel).
#pragma once

#include <cstdlib>

#include "tron_device.cuh"
#include "tron_launch.h"

namespace tbdev {

// per-thread family evaluation (the DevFamily expressions of tron_device.cuh
// on one thread: same tb_families.h terms, same ascending sums)
template <int FAM, int D>
struct ThFam;

template <int D>
struct ThFam<TB_FAMILY_BRANCH, D> {
    tb_branch_ctx ctx;
    __device__ __forceinline__ void prepare(const double* x, const double* prm) { tb_branch_ctx_init(x, prm, D, &ctx); }
    __device__ __forceinline__ double f(const double* prm) const { return tb_br_f(&ctx, prm, D); }
    __device__ __forceinline__ double grad(const double*, int i) const { return tb_br_grad(&ctx, D, i); }
    __device__ __forceinline__ double hess(const double* prm, int i, int j) const { return tb_br_hess(&ctx, prm, D, i, j); }
};

template <int D>
struct ThFam<TB_FAMILY_NCVX, D> {
    double e[D], he[D], sn[D], cs[D];  // x - c, H (x - c), sin x, cos x
    static constexpr int NH = D * (D + 1) / 2;
    __device__ __forceinline__ void prepare(const double* x, const double* prm) {
        const double* c = prm + NH;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            e[i] = x[i] - c[i];
            tb_sincos(x[i], &sn[i], &cs[i]);
        }
#pragma unroll
        for (int i = 0; i < D; ++i) he[i] = tb_ncvx_he_i(x, prm, D, i);
    }
    __device__ __forceinline__ double f(const double* prm) const {
        const double* k = prm + NH + D;
        const double* a = k + D;
        double q = 0.0, quart = 0.0, s = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            const double e2 = e[i] * e[i];
            q += e[i] * he[i];
            quart += k[i] * (e2 * e2);
            s += a[i] * sn[i];
        }
        return (0.5 * q + 0.25 * quart) + s;
    }
    __device__ __forceinline__ double grad(const double* prm, int i) const {
        const double* k = prm + NH + D;
        const double* a = k + D;
        const double e3 = (e[i] * e[i]) * e[i];
        return (he[i] + k[i] * e3) + a[i] * cs[i];
    }
    __device__ __forceinline__ double hess(const double* prm, int i, int j) const {
        const double h = tb_ncvx_H(prm, D, i, j);
        if (i != j) return h;
        const double* k = prm + NH + D;
        const double* a = k + D;
        return (h + (3.0 * k[i]) * (e[i] * e[i])) - a[i] * sn[i];
    }
};

template <int D, int FAM = TB_FAMILY_BRANCH>
struct Th {
    static_assert(D <= 8, "thread form: small problems only");
    double A[D * D];  // column-major Hessian
    double L[D * D];  // factor (lower), column-major
    double rd[D];     // RN(1 / L(j,j)) of the current factor
    const double* prm;
    const tb_tron_config* cfg;
    double extrap;
    ThFam<FAM, D> fam;

    // ------------------------------------------------ dense.hpp BLAS (ordered)
    __device__ __forceinline__ static bool in(unsigned m, int i) { return (m >> i) & 1u; }
    __device__ __forceinline__ static double dot(const double* x, const double* y, unsigned m) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i)
            if (in(m, i)) s += x[i] * y[i];
        return s;
    }
    __device__ __forceinline__ static double nrm2(const double* x, unsigned m) { return sqrt(dot(x, x, m)); }
    // y = A[m, m] x (column sweep, zero-skip on x_j; every row computed)
    __device__ __forceinline__ void gemv(const double* x, unsigned m, double* y) const {
#pragma unroll
        for (int i = 0; i < D; ++i) y[i] = 0.0 * 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const double xj = 1.0 * (in(m, j) ? x[j] : 0.0);
            if (xj != 0.0) {
#pragma unroll
                for (int i = 0; i < D; ++i) y[i] += xj * A[i + j * D];
            }
        }
    }

    // ------------------------------------------------ tron.hpp primitives
    __device__ __forceinline__ static double clip(double x, double l, double u) {
        return tb_smin(tb_smax(x, l), u);
    }
    __device__ __forceinline__ static double gpstep(double x, double alpha, double w, double l, double u) {
        const double trial = x + alpha * w;
        if (trial < l) return l - x;
        if (trial > u) return u - x;
        return alpha * w;
    }
    __device__ __forceinline__ static void breakpt(const double* x, const double* w, const double* l,
                                                   const double* u, unsigned m, double& bmin, double& bmax) {
        bool any = false;
        double lo = CUDART_INF, hi = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            if (!in(m, i)) continue;
            double b = 0.0;
            bool has = false;
            if (x[i] < u[i] && w[i] > 0.0) { b = (u[i] - x[i]) / w[i]; has = true; }
            else if (x[i] > l[i] && w[i] < 0.0) { b = (l[i] - x[i]) / w[i]; has = true; }
            if (has && !isfinite(b)) has = false;
            if (has) {  // finite, > 0: min / max are order-free
                any = true;
                lo = b < lo ? b : lo;
                hi = b > hi ? b : hi;
            }
        }
        bmin = any ? lo : 0.0;
        bmax = any ? hi : 0.0;
    }
    __device__ __forceinline__ static double pgnorm(const double* x, const double* g, const double* l,
                                                    const double* u, int n) {
        double m = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            if (i >= n) continue;
            double pg = g[i];
            if (x[i] <= l[i]) pg = tb_smin(g[i], 0.0);
            else if (x[i] >= u[i]) pg = tb_smax(g[i], 0.0);
            double v = fabs(pg);
            if (isnan(v)) v = 0.0;
            m = v > m ? v : m;
        }
        return m;
    }
    // tron.hpp:167-176
    __device__ __forceinline__ static int trqsol(const double* x, const double* w, double delta, unsigned m,
                                                 double& sigma) {
        double ptx = 0.0, ptp = 0.0, xtx = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i)
            if (in(m, i)) {
                ptx += w[i] * x[i];
                ptp += w[i] * w[i];
                xtx += x[i] * x[i];
            }
        if (ptp == 0.0) return TB_STATUS_ZERO_DIRECTION;
        const double dsq = delta * delta;
        const double rad = sqrt(tb_smax(ptx * ptx + ptp * tb_smax(dsq - xtx, 0.0), 0.0));
        if (ptx > 0.0) sigma = (dsq - xtx) / (ptx + rad);
        else sigma = (rad - ptx) / ptp;
        return 0;
    }
    __device__ __forceinline__ double quad_model(const double* g, const double* s, unsigned m, double& gs) const {
        double as[D];
        gemv(s, m, as);
        double sas = 0.0;
        gs = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i)
            if (in(m, i)) {
                gs += g[i] * s[i];
                sas += s[i] * as[i];
            }
        return gs + 0.5 * sas;
    }

    // ------------------------------------------------ dense.hpp:182-201 ccf
    // column j's quotients col[i] / d as Markstein quotients from one
    // RN(1/d) (tron_device.cuh quot: correctly rounded, bits of the division);
    // a column that met an out-of-range quotient is redone with IEEE divisions
    __device__ __forceinline__ bool chol(unsigned F, double sh) {
#pragma unroll
        for (int j = 0; j < D; ++j) {
            if (!in(F, j)) continue;
            double col[D];
#pragma unroll
            for (int i = j; i < D; ++i) {
                if (!in(F, i)) continue;
                double lij = A[i + j * D];
                if (i == j) lij += sh;
#pragma unroll
                for (int k = 0; k < j; ++k) {
                    if (!in(F, k)) continue;
                    const double ljk = L[j + k * D];
                    if (ljk != 0.0) lij -= ljk * L[i + k * D];
                }
                col[i] = lij;
            }
            const double pivot = col[j];
            if (!(pivot > 0.0)) return false;
            const double d = sqrt(pivot);
            const double r = __drcp_rn(d);
            L[j + j * D] = d;
            rd[j] = r;
            bool bad = false;
#pragma unroll
            for (int i = j + 1; i < D; ++i)
                if (in(F, i)) L[i + j * D] = quot<false>(col[i], d, r, bad);
            if (bad) {
#pragma unroll
                for (int i = j + 1; i < D; ++i)
                    if (in(F, i)) L[i + j * D] = col[i] / d;
            }
        }
        return true;
    }
    // Factor memo: ccf is a pure function of (A[F,F]); while the Hessian is
    // unchanged (rejected steps) and the free set repeats -- the stagnating
    // tail of a solve -- the previous factor is the reference's result again
    // (its shift attempts replay identically), so it is reused.
    unsigned memo_F = 0;
    bool memo_ok = false;
    __device__ __forceinline__ int ccf(unsigned F) {
#ifndef TB_CCF_MEMO
#define TB_CCF_MEMO 1
#endif
        if (TB_CCF_MEMO && memo_ok && F == memo_F) return 0;
        const int rc = ccf_compute(F);
        memo_ok = TB_CCF_MEMO && rc == 0;
        memo_F = F;
        return rc;
    }
    __device__ __forceinline__ int ccf_compute(unsigned F) {
        double max_diag = 0.0, max_abs = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            if (!in(F, i)) continue;
            double dg = fabs(A[i + i * D]);
            if (isnan(dg)) dg = 0.0;
            max_diag = dg > max_diag ? dg : max_diag;
#pragma unroll
            for (int j = 0; j < D; ++j) {
                if (!in(F, j)) continue;
                const double v = fabs(A[i + j * D]);
                if (!isnan(v)) max_abs = fmax(max_abs, v);
            }
        }
        const double alpha0 = tb_smax(1e-3 * max_diag, 1e-8);
        const double cap = 1e8 * tb_smax(1.0, max_abs);
        double sh = 0.0;
#pragma unroll 1
        for (int k = 0; k < 4096; ++k) {
            if (k > 0 && !(sh <= cap)) return TB_STATUS_FACTORIZATION_FAILED;
            if (chol(F, sh)) return 0;
            sh = tb_smax(2.0 * sh, alpha0);
        }
        return TB_STATUS_FACTORIZATION_FAILED;
    }
    // dense.hpp:224-228 / 229-235 on F (entries outside F: forward 0, backward pass-through)
    // quotients by L(i,i) from the stored RN(1/L(i,i)); one range test per
    // solve, a solve that met an out-of-range quotient reruns with IEEE
    template <bool IEEE>
    __device__ __forceinline__ bool trsv_fwd_q(const double* b, unsigned F, double* y) const {
        bool bad = false;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            if (!in(F, i)) {
                y[i] = 0.0;
                continue;
            }
            double s = b[i];
#pragma unroll
            for (int j = 0; j < i; ++j)
                if (in(F, j)) s -= L[i + j * D] * y[j];
            y[i] = quot<IEEE>(s, L[i + i * D], rd[i], bad);
        }
        return bad;
    }
    template <bool IEEE>
    __device__ __forceinline__ bool trsv_bwd_q(const double* b, unsigned F, double* y) const {
        bool bad = false;
#pragma unroll
        for (int i = D - 1; i >= 0; --i) {
            if (!in(F, i)) {
                y[i] = b[i];
                continue;
            }
            double s = b[i];
#pragma unroll
            for (int j = i + 1; j < D; ++j)
                if (in(F, j)) s -= L[j + i * D] * y[j];
            y[i] = quot<IEEE>(s, L[i + i * D], rd[i], bad);
        }
        return bad;
    }
    // dense.hpp:224-228 / 229-235 on F (entries outside F: forward 0, backward pass-through)
    __device__ __forceinline__ void trsv_fwd(const double* b, unsigned F, double* y) const {
        if (trsv_fwd_q<false>(b, F, y)) trsv_fwd_q<true>(b, F, y);
    }
    __device__ __forceinline__ void trsv_bwd(const double* b, unsigned F, double* y) const {
        if (trsv_bwd_q<false>(b, F, y)) trsv_bwd_q<true>(b, F, y);
    }

    // ------------------------------------------------ tron.hpp:290-344 PCG
    __device__ __forceinline__ int precond_cg(unsigned F, int nf, const double* gfree, double delta, double* step,
                                              int& cg_status, int& iters) {
        double w[D], r[D], p[D], z[D], q[D], t[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            w[i] = 0.0;
            t[i] = gfree[i] * -1.0;
        }
        trsv_fwd(t, F, r);  // bhat
        const double bnorm = nrm2(r, F);
        iters = 0;
        if (bnorm == 0.0) {
#pragma unroll
            for (int i = 0; i < D; ++i) step[i] = 0.0;
            cg_status = 0;
            return 0;
        }
#pragma unroll
        for (int i = 0; i < D; ++i) p[i] = r[i];
        double rho = dot(r, r, F);
        cg_status = 3;
#pragma unroll 1
        for (int k = 1; k <= nf; ++k) {
            iters = k;
            trsv_bwd(p, F, z);
            gemv(z, F, t);
            trsv_fwd(t, F, q);
            const double ptq = dot(p, q, F);
            double sigma;
            const int rc = trqsol(w, p, delta, F, sigma);
            if (rc) return rc;
            if (ptq <= 0.0) {
#pragma unroll
                for (int i = 0; i < D; ++i) w[i] += sigma * p[i];
                cg_status = 2;
                break;
            }
            const double alpha = rho / ptq;
            if (alpha >= sigma) {
#pragma unroll
                for (int i = 0; i < D; ++i) w[i] += sigma * p[i];
                cg_status = 1;
                break;
            }
#pragma unroll
            for (int i = 0; i < D; ++i) {
                w[i] += alpha * p[i];
                r[i] += (-alpha) * q[i];
            }
            const double rtr = dot(r, r, F);
            if (sqrt(rtr) <= cfg->cg_tol * bnorm) {
                cg_status = 0;
                break;
            }
            const double beta = rtr / rho;
#pragma unroll
            for (int i = 0; i < D; ++i) {
                p[i] = beta * p[i];
                p[i] += 1.0 * r[i];
            }
            rho = rtr;
        }
        trsv_bwd(w, F, step);
        return 0;
    }

    // tron.hpp:354-374 on the free set (all components computed, F ones used)
    __device__ __forceinline__ void line_search(const double* x, const double* l, const double* u, const double* g,
                                                const double* w, unsigned F, double* xn) const {
        const double kBetaFloor = 1e-12;
        double beta = 1.0;
        double bmin, bmax;
        breakpt(x, w, l, u, F, bmin, bmax);
        bool search = true;
#pragma unroll 1
        while (search && beta > bmin && beta > kBetaFloor) {
            double s[D];
#pragma unroll
            for (int i = 0; i < D; ++i) s[i] = gpstep(x[i], beta, w[i], l[i], u[i]);
            double gs;
            const double q = quad_model(g, s, F, gs);
            if (q <= cfg->mu0 * gs) search = false;
            else beta *= cfg->interp_factor;
        }
        if (beta < 1.0 && beta < bmin) beta = bmin;
#pragma unroll
        for (int i = 0; i < D; ++i) xn[i] = clip(x[i] + beta * w[i], l[i], u[i]);
    }

    // tron.hpp:201-250 (the warp kernel's single-trial-site state machine)
    __device__ __forceinline__ int cauchy(const double* x, const double* g, const double* l, const double* u,
                                          unsigned m, double delta, double alpha_start, double& alpha_out,
                                          double* s) const {
        const double radius = cfg->mu1 * delta;
        double alpha = alpha_start;
        double mg[D];
#pragma unroll
        for (int i = 0; i < D; ++i) mg[i] = -1.0 * g[i];
        double bmin, bmax;
        breakpt(x, mg, l, u, m, bmin, bmax);
        int mode = 0;  // 0 initial test, 1 interpolate, 2 extrapolate
        double alpha_good = alpha;
#pragma unroll 1
        for (;;) {
#pragma unroll
            for (int i = 0; i < D; ++i) s[i] = gpstep(x[i], -alpha, g[i], l[i], u[i]);
            const double nr = nrm2(s, m);
            const bool evalq = mode == 0 ? !(nr > radius) : (nr <= radius);
            bool qge = false;
            if (evalq) {
                double gs;
                const double q = quad_model(g, s, m, gs);
                if (!isfinite(q)) return TB_STATUS_EVALUATION_ERROR;
                qge = q >= cfg->mu0 * gs;
            }
            if (mode == 0) {
                if (!evalq || qge) {
                    mode = 1;
                    if (!(alpha > 1e-30)) break;
                    alpha *= cfg->interp_factor;
                    continue;
                }
                mode = 2;
                alpha_good = alpha;
                if (!(alpha <= bmax)) break;
                alpha *= extrap;
                continue;
            }
            if (mode == 1) {
                const bool search = evalq ? qge : true;
                if (!search || !(alpha > 1e-30)) break;
                alpha *= cfg->interp_factor;
                continue;
            }
            if (evalq && !qge) {
                alpha_good = alpha;
                if (!(alpha <= bmax)) break;
                alpha *= extrap;
                continue;
            }
            break;
        }
        if (mode == 2) {
            alpha = alpha_good;
#pragma unroll
            for (int i = 0; i < D; ++i) s[i] = gpstep(x[i], -alpha, g[i], l[i], u[i]);
        }
        alpha_out = alpha;
        return 0;
    }

    // tron.hpp:394-447
    __device__ __forceinline__ int subspace_step(const double* x0, const double* g, const double* l, const double* u,
                                                 int n, double delta, const double* cs, double* xout, double* s,
                                                 long long& cg_total) {
        const unsigned act = (1u << n) - 1u;
        double w[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            xout[i] = clip(x0[i] + 1.0 * cs[i], l[i], u[i]);
            s[i] = xout[i] - x0[i];
        }
        gemv(s, act, w);
        cg_total = 0;
#pragma unroll 1
        for (int faces = 0; faces < n; ++faces) {
            unsigned F = 0;
#pragma unroll
            for (int i = 0; i < D; ++i)
                if (i < n && l[i] < xout[i] && xout[i] < u[i]) F |= 1u << i;
            const int nf = __popc(F);
            if (nf == 0) break;
            int rc = ccf(F);
            if (rc) return rc;
#pragma unroll
            for (int i = 0; i < D; ++i)
                if (in(F, i) && L[i + i * D] == 0.0) return TB_STATUS_SINGULAR_FACTOR;
            double gfree[D], step[D], xn[D];
#pragma unroll
            for (int i = 0; i < D; ++i) gfree[i] = w[i] + g[i];
            const double gfnorm = nrm2(g, F);
            int cgs, its;
            rc = precond_cg(F, nf, gfree, delta, step, cgs, its);
            if (rc) return rc;
            cg_total += its;
            line_search(xout, l, u, gfree, step, F, xn);
#pragma unroll
            for (int i = 0; i < D; ++i)
                if (in(F, i)) {
                    s[i] += xn[i] - xout[i];
                    xout[i] = xn[i];
                }
            gemv(s, act, w);
            double gfnormf = 0.0;
#pragma unroll
            for (int i = 0; i < D; ++i)
                if (in(F, i)) {
                    const double t = w[i] + g[i];
                    gfnormf += t * t;
                }
            if (sqrt(gfnormf) <= cfg->cg_tol * gfnorm) break;
            if (cgs == 1 || cgs == 3) break;
        }
        return 0;
    }
};

// tron.hpp:453-549 solve() of problem `pid` by the calling thread (the warp
// kernel's loop structure: one evaluation site, fast-forward of the
// zero-change fixed point).
template <int D, int FAM = TB_FAMILY_BRANCH>
__device__ __forceinline__ void tron_solve_thread(const KernelArgs& a, const long long pid) {
    const unsigned long long t_start = globaltimer();
    Th<D, FAM> W;
    W.prm = a.prm + pid * a.stride;
    W.cfg = &a.cfg;
    W.extrap = a.extrap;
    const tb_tron_config& cfg = a.cfg;
    const int n = D;
    const unsigned act = (1u << n) - 1u;
    double l[D], u[D], x[D], xe[D], g[D], s[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
        l[i] = a.lo[pid * n + i];
        u[i] = a.up[pid * n + i];
        x[i] = a.x0[pid * n + i];
        g[i] = 0.0;
        s[i] = 0.0;
    }
    int status = TB_STATUS_ITER_LIMIT, iterations = 0;
    long long cg_iterations = 0, f_evals = 0;
    double f = 0.0, pg = 0.0;
    bool bad_bounds = false;
#pragma unroll
    for (int i = 0; i < D; ++i) bad_bounds |= !(l[i] <= u[i]);
    if (bad_bounds) {
        status = TB_STATUS_INVALID_BOUNDS;
    } else {
        const double kEta1 = 0.25, kEta2 = 0.75;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            x[i] = Th<D, FAM>::clip(x[i], l[i], u[i]);
            xe[i] = x[i];
        }
        double delta = 0.0, alpha_c = 1.0, delta_in = 0.0, alpha_in = 0.0;
        bool need_hessian = true;
        long long cg_its = 0;
#pragma unroll 1
        for (int iter = 0;; ++iter) {
            W.fam.prepare(xe, W.prm);
            const double fe = W.fam.f(W.prm);
            ++f_evals;
            bool take = iter == 0;
            if (iter > 0) {
                const double f_trial = fe;
                double as[D];
                W.gemv(s, act, as);
                double gs = 0.0, sas = 0.0, snn = 0.0;
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    gs += g[i] * s[i];
                    sas += s[i] * as[i];
                    snn += s[i] * s[i];
                }
                const double prered = -(gs + 0.5 * sas);
                const double actred = f - f_trial;
                const double snorm = sqrt(snn);
                if (iter == 1) delta = tb_smin(delta, snorm);
                double alphax;
                if (f_trial - f - gs <= 0.0) alphax = cfg.sigma3;
                else alphax = tb_smax(cfg.sigma1, -0.5 * (gs / (f_trial - f - gs)));
                if (actred < cfg.eta0 * prered)
                    delta = tb_smin(tb_smax(alphax, cfg.sigma1) * snorm, cfg.sigma2 * delta);
                else if (actred < kEta1 * prered)
                    delta = tb_smax(cfg.sigma1 * delta, tb_smin(alphax * snorm, cfg.sigma2 * delta));
                else if (actred < kEta2 * prered)
                    delta = tb_smax(cfg.sigma1 * delta, tb_smin(alphax * snorm, cfg.sigma3 * delta));
                else
                    delta = tb_smax(delta, tb_smin(alphax * snorm, cfg.sigma3 * delta));
                delta = tb_smin(delta, cfg.delta_max);
                take = actred > cfg.eta0 * prered;
                if (take) {
#pragma unroll
                    for (int i = 0; i < D; ++i) x[i] = xe[i];
                    f = f_trial;
                    need_hessian = true;
                }
            } else {
                f = fe;
            }
            if (take) {
#pragma unroll
                for (int i = 0; i < D; ++i) g[i] = W.fam.grad(W.prm, i);
                pg = Th<D, FAM>::pgnorm(x, g, l, u, n);
            }
            if (iter == 0) {
                delta = cfg.has_delta0 ? cfg.delta0 : tb_smax(Th<D, FAM>::nrm2(g, act), 1.0);
                status = pg <= cfg.tol_pg ? TB_STATUS_CONVERGED : TB_STATUS_ITER_LIMIT;
                if (status == TB_STATUS_CONVERGED) break;
            } else {
                if (take && pg <= cfg.tol_pg) {
                    status = TB_STATUS_CONVERGED;
                    break;
                }
                if (delta <= 1e-300) break;
                if (a.fast_forward && !take && iter >= 2 && delta == delta_in && alpha_c == alpha_in) {
                    const long long rem = cfg.max_iter - iter;
                    cg_iterations += rem * cg_its;
                    f_evals += rem;
                    iterations = cfg.max_iter;
                    break;
                }
            }
            if (iter + 1 > cfg.max_iter) break;
            iterations = iter + 1;
            if (need_hessian) {  // the context holds the current x
#pragma unroll
                for (int j = 0; j < D; ++j)
#pragma unroll
                    for (int i = j; i < D; ++i) {
                        const double h = W.fam.hess(W.prm, i, j);
                        W.A[i + j * D] = h;
                        W.A[j + i * D] = h;
                    }
                need_hessian = false;
                W.memo_ok = false;  // a new Hessian: the memoised factor is stale
            }
            delta_in = delta;
            alpha_in = alpha_c;
            double cs[D], alpha_new;
            int rc = W.cauchy(x, g, l, u, act, delta, alpha_c, alpha_new, cs);
            if (rc) {
                status = rc;
                break;
            }
            alpha_c = alpha_new;
            rc = W.subspace_step(x, g, l, u, n, delta, cs, xe, s, cg_its);
            if (rc) {
                status = rc;
                break;
            }
            cg_iterations += cg_its;
        }
    }
    if (a.x_star)
#pragma unroll
        for (int i = 0; i < D; ++i) a.x_star[pid * n + i] = x[i];
    if (a.f_star) a.f_star[pid] = f;
    if (a.pg_norm) a.pg_norm[pid] = pg;
    if (a.status) a.status[pid] = status;
    if (a.iterations) a.iterations[pid] = iterations;
    if (a.cg_iterations) a.cg_iterations[pid] = cg_iterations;
    if (a.f_evals) a.f_evals[pid] = f_evals;
    if (a.wall_time) a.wall_time[pid] = 1e-9 * (double)(globaltimer() - t_start);
}

// Routing (host): the thread form takes n = 4 batches (the whole batch or
// partition, not the concurrent chunk) of at least min_count problems: branch
// 4,096, ncvx 8,192 (KernelForm.THREAD forces it; round 2, with the factor
// memo: ncvx4 x8,192 0.471 vs 0.503 ms, x4,096 0.461 vs 0.363).  Round 1, device-
// resident, thread vs warp: ncvx d=4 x32,768 0.95 vs 1.40 ms, x20,467 0.83
// vs 0.97, x16,384 0.79 vs 0.81, x12,000 0.79 vs 0.66, x1,024 0.70 vs 0.30 (a
// lone problem's chain is slower on one thread); branch d=4 x65,536 1.12 vs
// 3.09, x20,467 0.81 vs 1.28, x4,096 0.43 vs 0.57.  At n = 6 / 8 the 255-register thread form loses (7.7 vs 7.4 ms
// branch6, 13.3 vs 3.6 ms ncvx8).  KernelForm.WARP forces the warp form.  Flop
// counting stays in the warp kernel.
template <int D, int FAM = TB_FAMILY_BRANCH, bool ORD = false>
__global__ void __launch_bounds__(64) tron_thread_kernel(const __grid_constant__ KernelArgs a) {
    const long long pid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (pid >= a.count || (a.skip && *a.skip)) return;
    tron_solve_thread<D, FAM>(a, ORD ? (long long)a.order[pid] : pid);  // ORD: ranked launch (tron_order.cu)
}

template <int D, int FAM>
inline cudaError_t launch_thread(const KernelArgs& a, cudaStream_t st) {
    const unsigned grid = (unsigned)((a.count + 63) / 64);
    if (a.order) tron_thread_kernel<D, FAM, true><<<grid, 64, 0, st>>>(a);
    else tron_thread_kernel<D, FAM><<<grid, 64, 0, st>>>(a);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace tbdev
