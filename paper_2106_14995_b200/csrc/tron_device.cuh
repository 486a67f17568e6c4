// tron_device.cuh — one warp solves one bound-constrained problem (d <= 32).
//
// Layout: lane i owns variable i.  Vectors (x, g, l, u, s, w, CG state) live
// in registers, one element per lane; the Hessian A and the shifted Cholesky
// factor L live in shared memory, column-major with leading dimension D
// (lane i reads A[i + j*D]: consecutive doubles, conflict-free).  Every
// scalar of the algorithm (f, delta, alpha, rho, ...) is computed redundantly
// and identically by all 32 lanes, so control flow is warp-uniform.
//
// The free-set sub-systems of subspace_step (tron.hpp:405-411: B = A[F,F],
// compacted) are NOT compacted: every routine takes a lane mask F and walks
// the free indices in ascending order (set-bit iteration), which reproduces
// the compacted loops operation for operation.
//
// Exact mode (nvcc --fmad=false): every reduction whose order matters is
// summed sequentially in ascending index order exactly like dense.hpp:79-84
// (dot) and dense.hpp:230-234 (backward solve); min/max and counting
// reductions (order-independent for the values they see) use warp shuffles.
// Results are bit-identical to the reference compiled with -ffp-contract=off.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "../../include/tb_capi.h"
#include "tb_families.h"
#include "tb_flops.h"

namespace tbdev {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ bool in_mask(unsigned m, int i) { return (m >> i) & 1u; }
__device__ __forceinline__ int low_bit(unsigned m) { return __ffs(m) - 1; }
__device__ __forceinline__ int high_bit(unsigned m) { return 31 - __clz(m); }

struct KernelArgs {
    int n;
    int nparams;
    long long count;
    long long stride;
    const double* x0;
    const double* lo;
    const double* up;
    const double* prm;
    tb_tron_config cfg;
    int fast_forward;
    double* x_star;
    double* f_star;
    double* pg_norm;
    int32_t* status;
    int32_t* iterations;
    int64_t* cg_iterations;
    int64_t* f_evals;
    double* wall_time;
    int64_t* flops;
};

// shared memory per warp (doubles)
template <int D>
struct SmemLayout {
    static constexpr int A = 0;                 // D*D Hessian
    static constexpr int L = A + D * D;         // D*D factor
    static constexpr int BUF = L + D * D;       // 2*D ordered-sum staging (double buffered)
    static constexpr int BB = BUF + 2 * D;      // D backward-solve results / second staging
    static constexpr int XS = BB + D;           // D point for family evaluations
    static constexpr int CTX = XS + D;          // family context (branch: sizeof(tb_branch_ctx))
    static constexpr int CTX_DOUBLES = (int)(sizeof(tb_branch_ctx) / sizeof(double));
    static constexpr int PRM = CTX + CTX_DOUBLES;  // staged parameters
    static constexpr int fixed() { return PRM; }
};

// ---------------------------------------------------------------- per warp
template <int D>
struct Warp {
    double* A;
    double* L;
    double* buf;  // 2*D
    double* bb;   // D
    double* xs;   // D
    const double* prm;
    const tb_tron_config* cfg;
    int n;
    int lane;
    int tog;        // ordered-sum buffer toggle (0 or D)
    unsigned act;   // lanes 0..n-1
    long long fl;   // algorithmic flop counter (tb_flops.h model)

    // ------------------------------------------------ ordered reductions
    // sum_{j in m, ascending} v_j, starting from 0.0 (dense.hpp:81-83).
    // Double-buffered staging: one __syncwarp per sum (the other buffer's
    // readers are ordered by the previous sum's barrier).
    __device__ __forceinline__ double seq_sum(double v, unsigned m) {
        double* b = buf + tog;
        tog ^= D;
        if (lane < D) b[lane] = v;
        __syncwarp();
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j)
            if (in_mask(m, j)) s += b[j];
        return s;
    }
    // two/three independent ordered sums (same bits as separate calls)
    __device__ __forceinline__ void seq_sum2(double a, double c, unsigned m, double& sa, double& sc) {
        double* b = buf + tog;
        tog ^= D;
        double* b2 = bb;
        if (lane < D) {
            b[lane] = a;
            b2[lane] = c;
        }
        __syncwarp();
        sa = 0.0;
        sc = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j)
            if (in_mask(m, j)) {
                sa += b[j];
                sc += b2[j];
            }
        __syncwarp();  // bb is not double buffered
    }
    __device__ __forceinline__ void seq_sum3(double a, double c, double e, unsigned m, double& sa, double& sc,
                                             double& se) {
        seq_sum2(a, c, m, sa, sc);
        se = seq_sum(e, m);
    }
    __device__ __forceinline__ double dot(double x, double y, unsigned m) {
        fl += 2 * __popc(m);
        return seq_sum(x * y, m);
    }
    __device__ __forceinline__ double nrm2(double x, unsigned m) {
        fl += 1;
        return sqrt(dot(x, x, m));
    }
    __device__ __forceinline__ double wmax(double v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
        return v;
    }
    __device__ __forceinline__ double wmin(double v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
        return v;
    }
    __device__ __forceinline__ double bcast(double v, int src) { return __shfl_sync(FULL, v, src); }

    // y = A[m,m] x over the lanes in m; dense.hpp:104-112 (alpha=1, beta=0):
    // column sweep j ascending, zero-skip on x_j.
    __device__ __forceinline__ double gemv(double x, unsigned m) {
        double* b = buf + tog;
        tog ^= D;
        if (lane < D) b[lane] = x;
        __syncwarp();
        const int nm = __popc(m);
        double y = 0.0 * 0.0;
        int used = 0;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            if (!in_mask(m, j)) continue;
            const double xj = 1.0 * b[j];
            if (xj == 0.0) continue;
            y += xj * A[lane + j * D];
            ++used;
        }
        fl += 2 * nm * used;
        return y;
    }

    // ------------------------------------------------ tron.hpp primitives
    __device__ __forceinline__ double clip(double x, double l, double u) { return tb_smin(tb_smax(x, l), u); }
    // tron.hpp:129-138
    __device__ __forceinline__ double gpstep(double x, double alpha, double w, double l, double u, unsigned m) {
        fl += 2 * __popc(m);
        const double trial = x + alpha * w;
        if (trial < l) return l - x;
        if (trial > u) return u - x;
        return alpha * w;
    }
    // tron.hpp:147-164 (min/max over finite breakpoints are order-free)
    __device__ __forceinline__ void breakpt(double x, double w, double l, double u, unsigned m, double& bmin,
                                            double& bmax) {
        fl += 2 * __popc(m);
        double b = 0.0;
        bool has = false;
        if (in_mask(m, lane)) {
            if (x < u && w > 0.0) { b = (u - x) / w; has = true; }
            else if (x > l && w < 0.0) { b = (l - x) / w; has = true; }
            if (has && !isfinite(b)) has = false;
        }
        if (!__any_sync(FULL, has)) {
            bmin = 0.0;
            bmax = 0.0;
            return;
        }
        bmin = wmin(has ? b : CUDART_INF);
        bmax = wmax(has ? b : -CUDART_INF);
    }
    // tron.hpp:112-121: inf-norm of the projected gradient; NaN components are
    // ignored by std::max, so they contribute 0
    __device__ __forceinline__ double pgnorm(double x, double g, double l, double u) {
        double pg = g;
        if (x <= l) pg = tb_smin(g, 0.0);
        else if (x >= u) pg = tb_smax(g, 0.0);
        double v = fabs(pg);
        if (!(lane < n) || isnan(v)) v = 0.0;
        return wmax(v);
    }
    // tron.hpp:167-176.  Returns 0 or TB_STATUS_ZERO_DIRECTION.
    __device__ __forceinline__ int trqsol(double x, double w, double delta, unsigned m, double& sigma) {
        double ptx, ptp, xtx;
        seq_sum3(w * x, w * w, x * x, m, ptx, ptp, xtx);
        fl += 6 * __popc(m) + 8;
        if (ptp == 0.0) return TB_STATUS_ZERO_DIRECTION;
        const double dsq = delta * delta;
        const double rad = sqrt(tb_smax(ptx * ptx + ptp * tb_smax(dsq - xtx, 0.0), 0.0));
        if (ptx > 0.0) sigma = (dsq - xtx) / (ptx + rad);
        else sigma = (rad - ptx) / ptp;
        return 0;
    }
    // tron.hpp:185-188: q(s) = g's + 0.5 s'As; also returns g's
    __device__ __forceinline__ double quad_model(double g, double s, unsigned m, double& gs) {
        const double as = gemv(s, m);
        double sas;
        seq_sum2(g * s, s * as, m, gs, sas);
        fl += 4 * __popc(m) + 2;
        return gs + 0.5 * sas;
    }

    // ------------------------------------------------ dense.hpp factorization
    // dense.hpp:138-156 on A[F,F]: left-looking, zero-skip on L(j,k), pivot
    // test !(pivot > 0), divide by sqrt(pivot).  Lane i keeps L(i,j) of the
    // current column in a register.
    __device__ __forceinline__ bool chol_left(unsigned F, int nf, double shift) {
        const bool inF = in_mask(F, lane);
        int rem = nf;  // free rows at or below the current column
#pragma unroll 1
        for (unsigned mj = F; mj; mj &= mj - 1) {
            const int j = low_bit(mj);
            const bool row = inF && lane >= j;
            double lij = row ? A[lane + j * D] : 0.0;
            if (lane == j) lij += shift;
            long long cnt = 0;
#pragma unroll 1
            for (unsigned mk = F & ((1u << j) - 1u); mk; mk &= mk - 1) {
                const int k = low_bit(mk);
                const double ljk = L[j + k * D];
                if (ljk == 0.0) continue;
                if (row) lij -= ljk * L[lane + k * D];
                ++cnt;
            }
            fl += 1 + 2 * rem * cnt;
            const double pivot = bcast(lij, j);
            if (!(pivot > 0.0)) return false;
            const double d = sqrt(pivot);
            if (lane == j) lij = d;
            else if (row) lij = lij / d;
            if (row) L[lane + j * D] = lij;
            fl += rem;  // sqrt + (rem - 1) divisions
            --rem;
            __syncwarp();
        }
        return true;
    }
    // dense.hpp:182-201 shifted_factorize.  Returns 0 or
    // TB_STATUS_FACTORIZATION_FAILED.
    __device__ __forceinline__ int ccf(unsigned F, int nf, double& shift) {
        const bool inF = in_mask(F, lane);
        double dg = inF ? fabs(A[lane + lane * D]) : 0.0;
        if (isnan(dg)) dg = 0.0;
        double ma = 0.0;
#pragma unroll 1
        for (unsigned mj = F; mj; mj &= mj - 1) {
            const double v = fabs(A[lane + low_bit(mj) * D]);
            if (inF && !isnan(v)) ma = fmax(ma, v);
        }
        const double max_diag = wmax(dg);
        const double max_abs = wmax(ma);
        const double alpha0 = tb_smax(1e-3 * max_diag, 1e-8);
        const double cap = 1e8 * tb_smax(1.0, max_abs);
        double alpha = 0.0;
#pragma unroll 1
        for (;;) {
            if (chol_left(F, nf, alpha)) {
                shift = alpha;
                return 0;
            }
            alpha = tb_smax(2.0 * alpha, alpha0);
            fl += 1;
            if (!(alpha <= cap)) return TB_STATUS_FACTORIZATION_FAILED;
        }
    }
    // dense.hpp:224-228 forward solve L b = rhs on F (column sweep == the
    // reference's ascending row dot-form, element by element)
    __device__ __forceinline__ double trsv_fwd(double b, unsigned F, double ldiag) {
        const bool inF = in_mask(F, lane);
        double s = b;
#pragma unroll 1
        for (unsigned mj = F; mj; mj &= mj - 1) {
            const int j = low_bit(mj);
            if (lane == j) s = s / ldiag;
            const double bj = bcast(s, j);
            if (inF && lane > j) s -= L[lane + j * D] * bj;
        }
        return s;
    }
    // dense.hpp:229-235 backward solve L^T b = rhs on F, exact order: for i
    // descending, s = b_i - sum_{j > i ascending} L(j,i) b_j.
    __device__ __forceinline__ double trsv_bwd(double b, unsigned F) {
        double out = b;
#pragma unroll 1
        for (unsigned mi = F; mi; mi &= ~(1u << high_bit(mi))) {
            const int i = high_bit(mi);
            double s = bcast(b, i);
#pragma unroll 1
            for (unsigned mj = F & ~((2u << i) - 1u); mj; mj &= mj - 1) {
                const int j = low_bit(mj);
                s -= L[j + i * D] * bb[j];
            }
            const double bi = s / L[i + i * D];
            if (lane == i) {
                out = bi;
                bb[i] = bi;
            }
            __syncwarp();
        }
        return out;
    }

    // ------------------------------------------------ tron.hpp:290-344
    // Steihaug PCG on the free set.  Returns 0 or an error status.
    // cg_status: 0 Converged, 1 Boundary, 2 NegCurve, 3 IterCap
    __device__ __forceinline__ int precond_cg(unsigned F, int nf, double gfree, double delta, double ldiag,
                                              double& step, int& cg_status, int& iters) {
        const long long nf2 = (long long)nf * nf;
        double w = 0.0;
        fl += nf;
        const double bhat = trsv_fwd(gfree * -1.0, F, ldiag);
        fl += nf2;
        const double bnorm = nrm2(bhat, F);
        iters = 0;
        if (bnorm == 0.0) {
            step = 0.0;
            cg_status = 0;
            return 0;
        }
        double r = bhat, p = r;
        double rho = dot(r, r, F);
        cg_status = 3;
#pragma unroll 1
        for (int k = 1; k <= nf; ++k) {
            iters = k;
            const double z = trsv_bwd(p, F);
            double q = gemv(z, F);
            q = trsv_fwd(q, F, ldiag);
            fl += 2 * nf2;
            const double ptq = dot(p, q, F);
            if (ptq <= 0.0) {
                double sigma;
                const int rc = trqsol(w, p, delta, F, sigma);
                if (rc) return rc;
                w += sigma * p;
                fl += 2 * nf;
                cg_status = 2;
                break;
            }
            const double alpha = rho / ptq;
            double sigma;
            const int rc = trqsol(w, p, delta, F, sigma);
            if (rc) return rc;
            fl += 1;
            if (alpha >= sigma) {
                w += sigma * p;
                fl += 2 * nf;
                cg_status = 1;
                break;
            }
            w += alpha * p;
            r += (-alpha) * q;
            fl += 4 * nf;
            const double rtr = dot(r, r, F);
            fl += 2;
            if (sqrt(rtr) <= cfg->cg_tol * bnorm) {
                cg_status = 0;
                break;
            }
            const double beta = rtr / rho;  // tron.hpp:335 scal then axpy
            p = beta * p;
            p += 1.0 * r;
            fl += 3 * nf + 1;
            rho = rtr;
        }
        step = trsv_bwd(w, F);
        fl += nf2;
        return 0;
    }

    // tron.hpp:354-374 on the free set
    __device__ __forceinline__ double line_search(double x, double l, double u, double g, double w, unsigned F) {
        const double kBetaFloor = 1e-12;
        double beta = 1.0;
        double bmin, bmax;
        breakpt(x, w, l, u, F, bmin, bmax);
        bool search = true;
#pragma unroll 1
        while (search && beta > bmin && beta > kBetaFloor) {
            const double s = gpstep(x, beta, w, l, u, F);
            double gs;
            const double q = quad_model(g, s, F, gs);
            fl += 2 * __popc(F) + 1;
            if (q <= cfg->mu0 * gs) search = false;
            else beta *= cfg->interp_factor;
        }
        if (beta < 1.0 && beta < bmin) beta = bmin;
        fl += 2 * __popc(F);
        return clip(x + beta * w, l, u);
    }

    // tron.hpp:201-250.  Returns 0 or TB_STATUS_EVALUATION_ERROR.
    __device__ __forceinline__ int cauchy(double x, double g, double l, double u, double delta, double alpha_start,
                                          double& alpha_out, double& s) {
        const unsigned m = act;
        const int nn = n;
        const double radius = cfg->mu1 * delta;
        const double extrap_factor = 1.0 / cfg->interp_factor;
        double alpha = alpha_start;
        const double mg = -1.0 * g;
        fl += nn;
        double bmin, bmax;
        breakpt(x, mg, l, u, m, bmin, bmax);
        s = gpstep(x, -alpha, g, l, u, m);
        bool interpolate;
        if (nrm2(s, m) > radius) {
            interpolate = true;
        } else {
            double gs;
            const double q = quad_model(g, s, m, gs);
            if (!isfinite(q)) return TB_STATUS_EVALUATION_ERROR;
            fl += 2 * nn + 1;
            interpolate = q >= cfg->mu0 * gs;
        }
        if (interpolate) {
            bool search = true;
#pragma unroll 1
            while (search && alpha > 1e-30) {
                alpha *= cfg->interp_factor;
                s = gpstep(x, -alpha, g, l, u, m);
                if (nrm2(s, m) <= radius) {
                    double gs;
                    const double q = quad_model(g, s, m, gs);
                    if (!isfinite(q)) return TB_STATUS_EVALUATION_ERROR;
                    fl += 2 * nn + 1;
                    search = q >= cfg->mu0 * gs;
                }
            }
        } else {
            double alpha_good = alpha;
            bool search = true;
#pragma unroll 1
            while (search && alpha <= bmax) {
                alpha *= extrap_factor;
                s = gpstep(x, -alpha, g, l, u, m);
                if (nrm2(s, m) <= radius) {
                    double gs;
                    const double q = quad_model(g, s, m, gs);
                    if (!isfinite(q)) return TB_STATUS_EVALUATION_ERROR;
                    fl += 2 * nn + 1;
                    if (q < cfg->mu0 * gs) alpha_good = alpha;
                    else search = false;
                } else {
                    search = false;
                }
            }
            alpha = alpha_good;
            s = gpstep(x, -alpha, g, l, u, m);
        }
        alpha_out = alpha;
        return 0;
    }

    // tron.hpp:394-447.  Returns 0 or an error status (factorization failure
    // is TB_STATUS_FACTORIZATION_FAILED, caught by solve like :499-501).
    __device__ __forceinline__ int subspace_step(double x0, double g, double l, double u, double delta, double cs,
                                                 double& xout, double& sout, long long& cg_total) {
        const int nn = n;
        xout = clip(x0 + 1.0 * cs, l, u);
        fl += 2 * nn;
        double s = xout - x0;
        fl += nn;
        double w = gemv(s, act);
        cg_total = 0;
#pragma unroll 1
        for (int faces = 0; faces < nn; ++faces) {
            const bool fr = lane < nn && l < xout && xout < u;
            const unsigned F = __ballot_sync(FULL, fr);
            const int nf = __popc(F);
            if (nf == 0) break;
            double shift;
            int rc = ccf(F, nf, shift);
            if (rc) return rc;
            const double ldiag = fr ? L[lane + lane * D] : 1.0;
            if (__any_sync(FULL, fr && ldiag == 0.0)) return TB_STATUS_SINGULAR_FACTOR;
            const double gfree = w + g;
            fl += nf;
            const double gfnorm = nrm2(g, F);
            double step;
            int cgs, its;
            rc = precond_cg(F, nf, gfree, delta, ldiag, step, cgs, its);
            if (rc) return rc;
            cg_total += its;
            const double xn = line_search(xout, l, u, gfree, step, F);
            if (fr) {
                s += xn - xout;
                xout = xn;
            }
            fl += 2 * nf;
            w = gemv(s, act);
            const double t = w + g;
            const double gfnormf = seq_sum(t * t, F);
            fl += 3 * nf + 2;
            if (sqrt(gfnormf) <= cfg->cg_tol * gfnorm) break;
            if (cgs == 1 || cgs == 3) break;
        }
        sout = s;
        return 0;
    }
};

// ------------------------------------------------------------ families
// Device evaluation of the families of tb_families.h.  prepare(x) builds the
// per-point context once (cooperatively across lanes); f / grad / hess at the
// same point reuse it.  The solver only ever evaluates grad and Hessian at the
// point of the most recent f evaluation (tron.hpp:474-476, 506, 532, 489),
// so one context per point suffices.  Each value is produced by the same
// tb_families.h expression as on the host.
template <int FAM, int D>
struct DevFamily {
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;  // per-lane caches
    tb_branch_ctx* ctx = nullptr;

    __device__ __forceinline__ void prepare(Warp<D>& W, double x) {
        const int lane = W.lane, n = W.n;
        const bool act = lane < n;
        if (act) W.xs[lane] = x;
        __syncwarp();
        const double* xs = W.xs;
        const double* prm = W.prm;
        if (FAM == TB_FAMILY_BOXQP) {
            if (act) {
                c0 = x - prm[(long)n * n + lane];    // d_i
                c1 = tb_boxqp_hd_i(xs, prm, n, lane); // (H d)_i
            }
        } else if (FAM == TB_FAMILY_NCVX) {
            if (act) {
                const double* c = prm + (long)n * (n + 1) / 2;
                c0 = x - c[lane];                    // e_i
                c1 = tb_ncvx_he_i(xs, prm, n, lane);  // (H e)_i
                tb_sincos(x, &c2, &c3);              // sin, cos
            }
        } else if (FAM == TB_FAMILY_BRANCH) {
            tb_branch_ctx* c = ctx;
            double b[8];
            tb_br_base(xs, b);
            if (lane < 8) c->base[lane] = b[lane];
            if (lane < 4) tb_br_flow(lane, b, prm, &c->F[lane], c->dF[lane], &c->cF[lane]);
            else if (lane < 6) {
                const int l = lane - 4;
                tb_br_volt(l, xs, prm, &c->rw[l], &c->cw[l], &c->rt[l], &c->ct[l]);
            }
            if (lane >= 8 && lane < 24) {
                const int e = lane - 8;
                tb_br_d2w(e / 4, e % 4, b, &c->d2wR[e], &c->d2wI[e]);
            }
            __syncwarp();
            if (lane < 2) {
                const int l = lane;
                if (n == 6) {
                    tb_br_line(l, xs, prm, c->F[2 * l], c->F[2 * l + 1], c->dF[2 * l], c->dF[2 * l + 1], &c->h[l],
                               &c->ch[l], c->dh[l]);
                } else {
                    c->h[l] = 0.0;
                    c->ch[l] = 0.0;
                    for (int k = 0; k < 4; ++k) c->dh[l][k] = 0.0;
                }
            }
            __syncwarp();
        }
    }
    __device__ __forceinline__ double f(Warp<D>& W) {
        const int lane = W.lane, n = W.n;
        const double* prm = W.prm;
        if (FAM == TB_FAMILY_HS45) return tb_hs45_f(W.xs, n);
        if (FAM == TB_FAMILY_BOXQP) return 0.5 * W.seq_sum(c0 * c1, W.act);
        if (FAM == TB_FAMILY_NCVX) {
            const double* k = prm + (long)n * (n + 1) / 2 + n;
            const double* a = k + n;
            const double e2 = c0 * c0;
            double q, quart, sn;
            const double kq = lane < n ? k[lane] * (e2 * e2) : 0.0;
            const double as = lane < n ? a[lane] * c2 : 0.0;
            W.seq_sum3(c0 * c1, kq, as, W.act, q, quart, sn);
            return (0.5 * q + 0.25 * quart) + sn;
        }
        return tb_br_f(ctx, prm, n);
    }
    __device__ __forceinline__ double grad(Warp<D>& W) {
        const int lane = W.lane, n = W.n;
        if (lane >= n) return 0.0;
        const double* prm = W.prm;
        if (FAM == TB_FAMILY_HS45) return tb_hs45_grad_i(W.xs, n, lane);
        if (FAM == TB_FAMILY_BOXQP) return c1;
        if (FAM == TB_FAMILY_NCVX) {
            const double* k = prm + (long)n * (n + 1) / 2 + n;
            const double* a = k + n;
            const double e3 = (c0 * c0) * c0;
            return (c1 + k[lane] * e3) + a[lane] * c3;
        }
        return tb_br_grad(ctx, n, lane);
    }
    // row `lane` of the Hessian into A[lane + j*D]
    __device__ __forceinline__ void hess(Warp<D>& W) {
        const int lane = W.lane, n = W.n;
        const double* prm = W.prm;
        if (lane < n) {
            if (FAM == TB_FAMILY_HS45) {
                for (int j = 0; j < n; ++j) W.A[lane + j * D] = tb_hs45_hess(W.xs, n, lane, j);
            } else if (FAM == TB_FAMILY_BOXQP) {
                for (int j = 0; j < n; ++j) W.A[lane + j * D] = tb_boxqp_hess(prm, n, lane, j);
            } else if (FAM == TB_FAMILY_NCVX) {
                const double* k = prm + (long)n * (n + 1) / 2 + n;
                const double* a = k + n;
                for (int j = 0; j < n; ++j) W.A[lane + j * D] = tb_ncvx_H(prm, n, lane, j);
                W.A[lane + lane * D] = (W.A[lane + lane * D] + (3.0 * k[lane]) * (c0 * c0)) - a[lane] * c2;
            } else {
                for (int j = 0; j < n; ++j) W.A[lane + j * D] = tb_br_hess(ctx, prm, n, lane, j);
            }
        }
        __syncwarp();
    }
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// tron.hpp:453-549 solve(), one problem per warp (one warp per block).
template <int FAM, int D>
__global__ void __launch_bounds__(32, 16) tron_solve_kernel(const __grid_constant__ KernelArgs a) {
    extern __shared__ double smem[];
    using SL = SmemLayout<D>;
    const long long pid = blockIdx.x;
    if (pid >= a.count) return;
    const unsigned long long t_start = globaltimer();

    Warp<D> W;
    W.A = smem + SL::A;
    W.L = smem + SL::L;
    W.buf = smem + SL::BUF;
    W.bb = smem + SL::BB;
    W.xs = smem + SL::XS;
    double* prm_s = smem + SL::PRM;
    W.n = a.n;
    W.lane = lane_id();
    W.tog = 0;
    W.act = (a.n >= 32) ? FULL : ((1u << a.n) - 1u);
    W.fl = 0;
    W.cfg = &a.cfg;
    const int n = a.n;
    const int lane = W.lane;
    const bool act = lane < n;
    const tb_tron_config& cfg = a.cfg;

    // stage this problem's parameters once (coalesced)
    if (a.prm) {
        const double* gp = a.prm + pid * a.stride;
        for (int k = lane; k < a.nparams; k += 32) prm_s[k] = gp[k];
    }
    W.prm = prm_s;
    DevFamily<FAM, D> fam;
    fam.ctx = reinterpret_cast<tb_branch_ctx*>(smem + SL::CTX);
    const double l = act ? a.lo[pid * n + lane] : 0.0;
    const double u = act ? a.up[pid * n + lane] : 0.0;
    double x = act ? a.x0[pid * n + lane] : 0.0;
    __syncwarp();

    int status = TB_STATUS_ITER_LIMIT;
    int iterations = 0;
    long long cg_iterations = 0, f_evals = 0;
    double f = 0.0, pg = 0.0;

    // tron.hpp:465-466
    if (__any_sync(FULL, act && !(l <= u))) {
        status = TB_STATUS_INVALID_BOUNDS;
    } else {
        const double kEta1 = 0.25, kEta2 = 0.75;
        x = W.clip(x, l, u);
        fam.prepare(W, x);
        f = fam.f(W);
        W.fl += tb_family_flops(FAM, n, 0);
        f_evals = 1;
        double g = fam.grad(W);
        W.fl += tb_family_flops(FAM, n, 1);
        pg = W.pgnorm(x, g, l, u);
        double delta = cfg.has_delta0 ? cfg.delta0 : tb_smax(W.nrm2(g, W.act), 1.0);
        double alpha_c = 1.0;
        bool need_hessian = true;
        status = pg <= cfg.tol_pg ? TB_STATUS_CONVERGED : TB_STATUS_ITER_LIMIT;

        if (status != TB_STATUS_CONVERGED) {
#pragma unroll 1
            for (int iter = 1; iter <= cfg.max_iter; ++iter) {
                iterations = iter;
                if (need_hessian) {  // family context holds the current x
                    fam.hess(W);
                    W.fl += tb_family_flops(FAM, n, 2);
                    need_hessian = false;
                }
                const long long fl_iter0 = W.fl;
                const double delta_in = delta, alpha_in = alpha_c;

                double cs, alpha_new;
                int rc = W.cauchy(x, g, l, u, delta, alpha_c, alpha_new, cs);
                if (rc) {
                    status = rc;
                    break;
                }
                alpha_c = alpha_new;
                double xt, s;
                long long cg_its;
                rc = W.subspace_step(x, g, l, u, delta, cs, xt, s, cg_its);
                if (rc) {
                    status = rc;  // FactorizationFailed caught like tron.hpp:499-501
                    break;
                }
                cg_iterations += cg_its;
                fam.prepare(W, xt);
                const double f_trial = fam.f(W);
                W.fl += tb_family_flops(FAM, n, 0);
                ++f_evals;

                const double as = W.gemv(s, W.act);
                double gs, sas, snn;
                W.seq_sum3(g * s, s * as, s * s, W.act, gs, sas, snn);
                W.fl += 6 * n + 1;
                const double prered = -(gs + 0.5 * sas);
                const double actred = f - f_trial;
                const double snorm = sqrt(snn);
                W.fl += 4;
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
                W.fl += 12;

                const bool accepted = actred > cfg.eta0 * prered;
                if (accepted) {
                    x = xt;
                    f = f_trial;
                    g = fam.grad(W);  // context was prepared at xt
                    W.fl += tb_family_flops(FAM, n, 1);
                    need_hessian = true;
                    pg = W.pgnorm(x, g, l, u);
                    if (pg <= cfg.tol_pg) {
                        status = TB_STATUS_CONVERGED;
                        break;
                    }
                }
                if (delta <= 1e-300) break;
                // Zero-change fixed point: a rejected
                // iteration k >= 2 that leaves delta and alpha_c bitwise
                // unchanged leaves the whole solver state (x, f, g, A, delta,
                // alpha_c) unchanged, so every remaining iteration replays it
                // exactly.  Fast-forward with identical counters.
                if (a.fast_forward && !accepted && iter >= 2 && delta == delta_in && alpha_c == alpha_in) {
                    const long long rem = cfg.max_iter - iter;
                    cg_iterations += rem * cg_its;
                    f_evals += rem;
                    W.fl += rem * (W.fl - fl_iter0);
                    iterations = cfg.max_iter;
                    break;
                }
            }
        }
    }

    if (act && a.x_star) a.x_star[pid * n + lane] = x;
    if (lane == 0) {
        if (a.f_star) a.f_star[pid] = f;
        if (a.pg_norm) a.pg_norm[pid] = pg;
        if (a.status) a.status[pid] = status;
        if (a.iterations) a.iterations[pid] = iterations;
        if (a.cg_iterations) a.cg_iterations[pid] = cg_iterations;
        if (a.f_evals) a.f_evals[pid] = f_evals;
        if (a.flops) a.flops[pid] = W.fl;
        if (a.wall_time) a.wall_time[pid] = 1e-9 * (double)(globaltimer() - t_start);
    }
}

}  // namespace tbdev
