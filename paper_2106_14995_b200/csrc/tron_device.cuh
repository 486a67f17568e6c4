// tron_device.cuh — one warp solves one bound-constrained problem (d <= 32).
//
// Layout: lane i owns variable i.  Vectors (x, g, l, u, s, w, CG state) live
// in registers, one element per lane; the Hessian A and the shifted Cholesky
// factor L live in shared memory, column-major with leading dimension D
// (lane i reads A[i + j*D]: consecutive doubles, conflict-free).  Every
// scalar of the algorithm (f, delta, alpha, rho, ...) is computed redundantly
// and identically by all 32 lanes, so control flow is warp-uniform.
//
// D is a compile-time bound (the exact dimension for the branch family, the
// next power of two otherwise); small-D kernels are fully unrolled.
//
// The free-set sub-systems of subspace_step (tron.hpp:405-411: B = A[F,F],
// compacted) are NOT compacted: every routine takes a lane mask F and walks
// the free indices in ascending order, which reproduces the compacted loops
// operation for operation.
//
// Exact mode (nvcc --fmad=false): every reduction whose order matters is
// summed sequentially in ascending index order exactly like dense.hpp:79-84
// (dot) and dense.hpp:230-234 (backward solve).  Ordered sums run over all D
// slots with +0.0 in the masked-out ones: a sum that starts at +0.0 and only
// adds can never be -0.0 (round-to-nearest), so s + 0.0 == s bit-for-bit and
// the padded sum equals the reference's sum over the free indices.  min/max
// and counting reductions (order-independent for the non-negative values they
// see) use integer warp reductions on the IEEE bit patterns.  Results are
// bit-identical to the reference compiled with -ffp-contract=off.
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

// max / min over the warp of NON-NEGATIVE doubles (+0.0 .. +inf, no NaN):
// IEEE bit patterns of such values order like unsigned integers.
__device__ __forceinline__ double warp_max_nonneg(double v) {
    const unsigned long long b = __double_as_longlong(v);
    const unsigned hi = __reduce_max_sync(FULL, (unsigned)(b >> 32));
    const unsigned lo = __reduce_max_sync(FULL, (unsigned)(b >> 32) == hi ? (unsigned)b : 0u);
    return __longlong_as_double((long long)(((unsigned long long)hi << 32) | lo));
}
__device__ __forceinline__ double warp_min_nonneg(double v) {
    const unsigned long long b = __double_as_longlong(v);
    const unsigned hi = __reduce_min_sync(FULL, (unsigned)(b >> 32));
    const unsigned lo = __reduce_min_sync(FULL, (unsigned)(b >> 32) == hi ? (unsigned)b : 0xffffffffu);
    return __longlong_as_double((long long)(((unsigned long long)hi << 32) | lo));
}

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

// shared memory per warp (doubles; every region starts at an even offset)
template <int D>
struct SmemLayout {
    static constexpr int A = 0;              // D*D Hessian
    static constexpr int L = A + D * D;      // D*D factor
    static constexpr int S1 = L + D * D;     // 2*D ordered-sum staging (double buffered)
    static constexpr int S2 = S1 + 2 * D;    // 2*D second staging (double buffered)
    static constexpr int XS = S2 + 2 * D;    // D point for family evaluations
    static constexpr int CTX = XS + D;       // family context (branch: sizeof(tb_branch_ctx))
    static constexpr int CTX_DOUBLES = (int)((sizeof(tb_branch_ctx) / sizeof(double) + 1) & ~1);
    static constexpr int PRM = CTX + CTX_DOUBLES;  // staged parameters
    static constexpr int fixed() { return PRM; }
    static_assert(D % 2 == 0, "D must be even (16-byte staging loads)");
};

// ---------------------------------------------------------------- per warp
template <int D, bool COUNT>
struct Warp {
    static constexpr bool kUnroll = D <= 8;
    double* A;
    double* L;
    double* s1;  // 2*D
    double* s2;  // 2*D
    double* xs;  // D
    const double* prm;
    const tb_tron_config* cfg;
    int n;
    int lane;
    int tog;        // staging toggle (0 or D)
    unsigned act;   // lanes 0..n-1
    long long fl;   // algorithmic flop counter (tb_flops.h model), COUNT builds only

    __device__ __forceinline__ void count(long long v) {
        if (COUNT) fl += v;
    }

    // ------------------------------------------------ ordered reductions
    // sum_{j in m, ascending} v_j from +0.0 (dense.hpp:81-83), zero-padded
    __device__ __forceinline__ double padded_sum(const double* b) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < D; j += 2) {
            const double2 t = *reinterpret_cast<const double2*>(b + j);
            s += t.x;
            s += t.y;
        }
        return s;
    }
    __device__ __forceinline__ double seq_sum(double v, unsigned m) {
        double* b = s1 + tog;
        tog ^= D;
        if (lane < D) b[lane] = in_mask(m, lane) ? v : 0.0;
        __syncwarp();
        return padded_sum(b);
    }
    // two independent ordered sums, one barrier
    __device__ __forceinline__ void seq_sum2(double a, double c, unsigned m, double& sa, double& sc) {
        double* b = s1 + tog;
        double* b2 = s2 + tog;
        tog ^= D;
        if (lane < D) {
            const bool in = in_mask(m, lane);
            b[lane] = in ? a : 0.0;
            b2[lane] = in ? c : 0.0;
        }
        __syncwarp();
        sa = padded_sum(b);
        sc = padded_sum(b2);
    }
    __device__ __forceinline__ void seq_sum3(double a, double c, double e, unsigned m, double& sa, double& sc,
                                             double& se) {
        seq_sum2(a, c, m, sa, sc);
        se = seq_sum(e, m);
    }
    __device__ __forceinline__ double dot(double x, double y, unsigned m) {
        count(2 * __popc(m));
        return seq_sum(x * y, m);
    }
    __device__ __forceinline__ double nrm2(double x, unsigned m) {
        count(1);
        return sqrt(dot(x, x, m));
    }
    __device__ __forceinline__ double bcast(double v, int src) { return __shfl_sync(FULL, v, src); }

    // y = A[m,m] x over the lanes in m; dense.hpp:104-112 (alpha=1, beta=0):
    // column sweep j ascending, zero-skip on x_j (masked columns staged as 0)
    __device__ __forceinline__ double gemv(double x, unsigned m) {
        double* b = s1 + tog;
        tog ^= D;
        if (lane < D) b[lane] = in_mask(m, lane) ? x : 0.0;
        __syncwarp();
        double y = 0.0 * 0.0;
        int used = 0;
        if (lane < D) {
#pragma unroll
            for (int j = 0; j < D; j += 2) {
                const double2 t = *reinterpret_cast<const double2*>(b + j);
                const double x0 = 1.0 * t.x, x1 = 1.0 * t.y;
                if (x0 != 0.0) {
                    y += x0 * A[lane + j * D];
                    ++used;
                }
                if (x1 != 0.0) {
                    y += x1 * A[lane + (j + 1) * D];
                    ++used;
                }
            }
        }
        if (COUNT) fl += 2LL * __popc(m) * __shfl_sync(FULL, used, 0);
        return y;
    }

    // ------------------------------------------------ tron.hpp primitives
    __device__ __forceinline__ double clip(double x, double l, double u) { return tb_smin(tb_smax(x, l), u); }
    // tron.hpp:129-138
    __device__ __forceinline__ double gpstep(double x, double alpha, double w, double l, double u, unsigned m) {
        count(2 * __popc(m));
        const double trial = x + alpha * w;
        if (trial < l) return l - x;
        if (trial > u) return u - x;
        return alpha * w;
    }
    // tron.hpp:147-164: breakpoints are finite and > 0 (x strictly inside the
    // bound it moves to), so min/max are order-free integer reductions
    __device__ __forceinline__ void breakpt(double x, double w, double l, double u, unsigned m, double& bmin,
                                            double& bmax) {
        count(2 * __popc(m));
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
        bmin = warp_min_nonneg(has ? b : CUDART_INF);
        bmax = warp_max_nonneg(has ? b : 0.0);
    }
    // tron.hpp:112-121: inf-norm of the projected gradient; NaN components are
    // ignored by std::max, so they contribute 0
    __device__ __forceinline__ double pgnorm(double x, double g, double l, double u) {
        double pg = g;
        if (x <= l) pg = tb_smin(g, 0.0);
        else if (x >= u) pg = tb_smax(g, 0.0);
        double v = fabs(pg);
        if (!(lane < n) || isnan(v)) v = 0.0;
        return warp_max_nonneg(v);
    }
    // tron.hpp:167-176.  Returns 0 or TB_STATUS_ZERO_DIRECTION.
    __device__ __forceinline__ int trqsol(double x, double w, double delta, unsigned m, double& sigma) {
        double ptx, ptp, xtx;
        seq_sum3(w * x, w * w, x * x, m, ptx, ptp, xtx);
        count(6 * __popc(m) + 8);
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
        count(4 * __popc(m) + 2);
        return gs + 0.5 * sas;
    }

    // ------------------------------------------------ dense.hpp factorization
    // one column of dense.hpp:141-154 (left-looking, zero-skip on L(j,k),
    // pivot test !(pivot > 0), division by sqrt(pivot))
    __device__ __forceinline__ bool chol_column(unsigned F, int j, double shift, int rem) {
        const bool row = in_mask(F, lane) && lane >= j;
        double lij = row ? A[lane + j * D] : 0.0;
        if (lane == j) lij += shift;
        long long cnt = 0;
        if (kUnroll) {
#pragma unroll
            for (int k = 0; k < D - 1; ++k) {
                if (k >= j || !in_mask(F, k)) continue;
                const double ljk = L[j + k * D];
                if (ljk == 0.0) continue;
                if (row) lij -= ljk * L[lane + k * D];
                ++cnt;
            }
        } else {
#pragma unroll 1
            for (unsigned mk = F & ((1u << j) - 1u); mk; mk &= mk - 1) {
                const int k = low_bit(mk);
                const double ljk = L[j + k * D];
                if (ljk == 0.0) continue;
                if (row) lij -= ljk * L[lane + k * D];
                ++cnt;
            }
        }
        count(1 + 2LL * rem * cnt);
        const double pivot = bcast(lij, j);
        if (!(pivot > 0.0)) return false;
        const double d = sqrt(pivot);
        const double q = lij / d;  // every lane (non-rows hold 0): no divergence
        lij = lane == j ? d : q;
        if (row) L[lane + j * D] = lij;
        count(rem);  // sqrt + (rem - 1) divisions
        __syncwarp();
        return true;
    }
    __device__ __forceinline__ bool chol_left(unsigned F, int nf, double shift) {
        int rem = nf;  // free rows at or below the current column
        if (kUnroll) {
#pragma unroll
            for (int j = 0; j < D; ++j) {
                if (!in_mask(F, j)) continue;
                if (!chol_column(F, j, shift, rem)) return false;
                --rem;
            }
        } else {
#pragma unroll 1
            for (unsigned mj = F; mj; mj &= mj - 1) {
                if (!chol_column(F, low_bit(mj), shift, rem)) return false;
                --rem;
            }
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
        if (inF) {
#pragma unroll 1
            for (unsigned mj = F; mj; mj &= mj - 1) {
                const double v = fabs(A[lane + low_bit(mj) * D]);
                if (!isnan(v)) ma = fmax(ma, v);
            }
        }
        const double max_diag = warp_max_nonneg(dg);
        const double max_abs = warp_max_nonneg(ma);
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
            count(1);
            if (!(alpha <= cap)) return TB_STATUS_FACTORIZATION_FAILED;
        }
    }
    // dense.hpp:224-228 forward solve L b = rhs on F (column sweep == the
    // reference's ascending row dot-form, element by element).  ldiag is 1
    // outside F so every lane divides benign operands (no divergence).
    __device__ __forceinline__ void trsv_fwd_step(int j, unsigned F, bool inF, double ldiag, double& s) {
        const double q = s / ldiag;
        const double bj = bcast(q, j);
        if (lane == j) s = q;
        else if (inF && lane > j) s -= L[lane + j * D] * bj;
    }
    __device__ __forceinline__ double trsv_fwd(double b, unsigned F, double ldiag) {
        const bool inF = in_mask(F, lane);
        double s = inF ? b : 0.0;
        if (kUnroll) {
#pragma unroll
            for (int j = 0; j < D; ++j)
                if (in_mask(F, j)) trsv_fwd_step(j, F, inF, ldiag, s);
        } else {
#pragma unroll 1
            for (unsigned mj = F; mj; mj &= mj - 1) trsv_fwd_step(low_bit(mj), F, inF, ldiag, s);
        }
        return s;
    }
    // dense.hpp:229-235 backward solve L^T b = rhs on F, exact order: for i
    // descending, s = b_i - sum_{j > i ascending} L(j,i) b_j.  Every lane
    // computes every b_i (redundantly, identical bits).
    __device__ __forceinline__ double trsv_bwd(double b, unsigned F) {
        double out = b;
        if (kUnroll) {
            double bv[D];
#pragma unroll
            for (int i = D - 1; i >= 0; --i) {
                bv[i] = 0.0;
                if (!in_mask(F, i)) continue;
                double s = bcast(b, i);
#pragma unroll
                for (int j = i + 1; j < D; ++j)
                    if (in_mask(F, j)) s -= L[j + i * D] * bv[j];
                bv[i] = s / L[i + i * D];
                if (lane == i) out = bv[i];
            }
        } else {
            double* bb = s2 + tog;  // dedicated staging for this solve
            tog ^= D;
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
        count(nf);
        const double bhat = trsv_fwd(gfree * -1.0, F, ldiag);
        count(nf2);
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
            count(2 * nf2);
            const double ptq = dot(p, q, F);
            if (ptq <= 0.0) {
                double sigma;
                const int rc = trqsol(w, p, delta, F, sigma);
                if (rc) return rc;
                w += sigma * p;
                count(2 * nf);
                cg_status = 2;
                break;
            }
            const double alpha = rho / ptq;
            double sigma;
            const int rc = trqsol(w, p, delta, F, sigma);
            if (rc) return rc;
            count(1);
            if (alpha >= sigma) {
                w += sigma * p;
                count(2 * nf);
                cg_status = 1;
                break;
            }
            w += alpha * p;
            r += (-alpha) * q;
            count(4 * nf);
            const double rtr = dot(r, r, F);
            count(2);
            if (sqrt(rtr) <= cfg->cg_tol * bnorm) {
                cg_status = 0;
                break;
            }
            const double beta = rtr / rho;  // tron.hpp:335 scal then axpy
            p = beta * p;
            p += 1.0 * r;
            count(3 * nf + 1);
            rho = rtr;
        }
        step = trsv_bwd(w, F);
        count(nf2);
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
            count(2 * __popc(F) + 1);
            if (q <= cfg->mu0 * gs) search = false;
            else beta *= cfg->interp_factor;
        }
        if (beta < 1.0 && beta < bmin) beta = bmin;
        count(2 * __popc(F));
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
        count(nn);
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
            count(2 * nn + 1);
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
                    count(2 * nn + 1);
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
                    count(2 * nn + 1);
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
        count(2 * nn);
        double s = xout - x0;
        count(nn);
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
            count(nf);
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
            count(2 * nf);
            w = gemv(s, act);
            const double t = w + g;
            const double gfnormf = seq_sum(t * t, F);
            count(3 * nf + 2);
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
template <int FAM, int D, bool COUNT>
struct DevFamily {
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;  // per-lane caches
    tb_branch_ctx* ctx = nullptr;

    __device__ __forceinline__ void prepare(Warp<D, COUNT>& W, double x) {
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
    __device__ __forceinline__ double f(Warp<D, COUNT>& W) {
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
    __device__ __forceinline__ double grad(Warp<D, COUNT>& W) {
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
    __device__ __forceinline__ void hess(Warp<D, COUNT>& W) {
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
template <int FAM, int D, bool COUNT>
__global__ void __launch_bounds__(32, 16) tron_solve_kernel(const __grid_constant__ KernelArgs a) {
    extern __shared__ double smem[];
    using SL = SmemLayout<D>;
    const long long pid = blockIdx.x;
    if (pid >= a.count) return;
    const unsigned long long t_start = globaltimer();

    Warp<D, COUNT> W;
    W.A = smem + SL::A;
    W.L = smem + SL::L;
    W.s1 = smem + SL::S1;
    W.s2 = smem + SL::S2;
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
    DevFamily<FAM, D, COUNT> fam;
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
        W.count(tb_family_flops(FAM, n, 0));
        f_evals = 1;
        double g = fam.grad(W);
        W.count(tb_family_flops(FAM, n, 1));
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
                    W.count(tb_family_flops(FAM, n, 2));
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
                W.count(tb_family_flops(FAM, n, 0));
                ++f_evals;

                const double as = W.gemv(s, W.act);
                double gs, sas, snn;
                W.seq_sum3(g * s, s * as, s * s, W.act, gs, sas, snn);
                W.count(6 * n + 1);
                const double prered = -(gs + 0.5 * sas);
                const double actred = f - f_trial;
                const double snorm = sqrt(snn);
                W.count(4);
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
                W.count(12);

                const bool accepted = actred > cfg.eta0 * prered;
                if (accepted) {
                    x = xt;
                    f = f_trial;
                    g = fam.grad(W);  // context was prepared at xt
                    W.count(tb_family_flops(FAM, n, 1));
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
                    W.count(rem * (W.fl - fl_iter0));
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
