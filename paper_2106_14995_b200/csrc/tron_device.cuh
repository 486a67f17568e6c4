// tron_device.cuh — one warp solves one bound-constrained problem (d <= 32).
//
// Layout: lane i owns variable i.  Vectors (x, g, l, u, s, w, CG state) live
// in registers, one element per lane; the Hessian A and the shifted Cholesky
// factor L live in shared memory, column-major with leading dimension D
// (lane i reads A[i + j*D]: 32 consecutive doubles, conflict-free).  Every
// scalar of the algorithm (f, delta, alpha, rho, ...) is computed redundantly
// and identically by all 32 lanes, so control flow is warp-uniform.
//
// The free-set sub-systems of subspace_step (tron.hpp:405-411: B = A[F,F],
// compacted) are NOT compacted: every routine takes a lane mask F and walks
// the free indices in ascending order, which reproduces the compacted loops
// operation for operation.
//
// Exact mode (the default build, nvcc --fmad=false): every reduction whose
// order matters is summed sequentially in ascending index order exactly like
// dense.hpp:79-84 (dot) and dense.hpp:230-234 (backward solve); min/max and
// counting reductions (order-independent for the values they see) use warp
// shuffles.  Results are bit-identical to the reference compiled with
// -ffp-contract=off.
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

// ---------------------------------------------------------------- per warp
template <int D>
struct Warp {
    // shared-memory work areas (set up by the kernel)
    double* A;    // D*D Hessian
    double* L;    // D*D shifted Cholesky factor of A[F,F] (original indexing)
    double* buf;  // D   staging for ordered sums / broadcasts
    double* bb;   // D   backward-solve results
    double* xs;   // D   point staged for family evaluations
    const double* prm;
    int n;
    int lane;
    unsigned act;      // lanes 0..n-1
    long long fl;      // algorithmic flop counter (tb_flops.h model)
    tb_tron_config cfg;

    // ------------------------------------------------ ordered reductions
    // sum_{j in m, ascending} v_j, starting from 0.0 (dense.hpp:81-83)
    __device__ __forceinline__ double seq_sum(double v, unsigned m) {
        if (lane < D) buf[lane] = v;
        __syncwarp();
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j)
            if (in_mask(m, j)) s += buf[j];
        __syncwarp();
        return s;
    }
    // three independent ordered sums in one pass (same bits as three calls)
    __device__ __forceinline__ void seq_sum3(double a, double b, double c, unsigned m, double& sa,
                                             double& sb, double& sc) {
        double* b2 = buf + 0;
        if (lane < D) {
            b2[lane] = a;
            bb[lane] = b;
        }
        __syncwarp();
        sa = 0.0;
        sb = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j)
            if (in_mask(m, j)) {
                sa += b2[j];
                sb += bb[j];
            }
        __syncwarp();
        if (lane < D) b2[lane] = c;
        __syncwarp();
        sc = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j)
            if (in_mask(m, j)) sc += b2[j];
        __syncwarp();
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
        if (lane < D) buf[lane] = x;
        __syncwarp();
        const int nm = __popc(m);
        double y = 0.0 * 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            if (!in_mask(m, j)) continue;
            const double xj = 1.0 * buf[j];
            if (xj == 0.0) continue;
            y += xj * A[lane + j * D];
            fl += 2 * nm;
        }
        __syncwarp();
        return y;
    }

    // ------------------------------------------------ tron.hpp primitives
    __device__ __forceinline__ double clip(double x, double l, double u) {
        return tb_smin(tb_smax(x, l), u);
    }
    // tron.hpp:129-138
    __device__ __forceinline__ double gpstep(double x, double alpha, double w, double l, double u,
                                             unsigned m) {
        fl += 2 * __popc(m);
        const double trial = x + alpha * w;
        if (trial < l) return l - x;
        if (trial > u) return u - x;
        return alpha * w;
    }
    // tron.hpp:147-164 (min/max over finite breakpoints are order-free)
    __device__ __forceinline__ void breakpt(double x, double w, double l, double u, unsigned m,
                                            int& count, double& bmin, double& bmax) {
        fl += 2 * __popc(m);
        double b = 0.0;
        bool has = false;
        if (in_mask(m, lane)) {
            if (x < u && w > 0.0) { b = (u - x) / w; has = true; }
            else if (x > l && w < 0.0) { b = (l - x) / w; has = true; }
            if (has && !isfinite(b)) has = false;
        }
        const unsigned hm = __ballot_sync(FULL, has);
        count = __popc(hm);
        if (count == 0) {
            bmin = 0.0;
            bmax = 0.0;
            return;
        }
        bmin = wmin(has ? b : CUDART_INF);
        bmax = wmax(has ? b : -CUDART_INF);
    }
    // tron.hpp:112-121: inf-norm of the projected gradient, NaN ignored by
    // std::max (so NaN lanes contribute 0)
    __device__ __forceinline__ double pgnorm(double x, double g, double l, double u) {
        double pg = g;
        if (x <= l) pg = tb_smin(g, 0.0);
        else if (x >= u) pg = tb_smax(g, 0.0);
        double v = fabs(pg);
        if (!(lane < n) || isnan(v)) v = 0.0;
        return wmax(v);
    }
    // tron.hpp:167-176.  Returns 0 or TB_STATUS_ZERO_DIRECTION.
    __device__ __forceinline__ int trqsol(double x, double w, double delta, unsigned m,
                                          double& sigma) {
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
        double sas, unused;
        seq_sum3(g * s, s * as, 0.0, m, gs, sas, unused);
        fl += 4 * __popc(m) + 2;
        return gs + 0.5 * sas;
    }

    // ------------------------------------------------ dense.hpp factorization
    // dense.hpp:138-156 on A[F,F]: left-looking, zero-skip on L(j,k), pivot
    // test !(pivot > 0), divide by sqrt(pivot).  Lane i keeps L(i,j) of the
    // current column in a register.
    __device__ __forceinline__ bool chol_left(unsigned F, int nf, double shift) {
        int jpos = 0;
#pragma unroll 1
        for (int j = 0; j < D; ++j) {
            if (!in_mask(F, j)) continue;
            const bool row = in_mask(F, lane) && lane >= j;
            double lij = row ? A[lane + j * D] : 0.0;
            if (lane == j) lij += shift;
            fl += 1;
#pragma unroll 1
            for (int k = 0; k < j; ++k) {
                if (!in_mask(F, k)) continue;
                const double ljk = L[j + k * D];
                if (ljk == 0.0) continue;
                if (row) lij -= ljk * L[lane + k * D];
                fl += 2 * (nf - jpos);
            }
            const double pivot = bcast(lij, j);
            if (!(pivot > 0.0)) return false;
            const double d = sqrt(pivot);
            if (lane == j) lij = d;
            else if (row) lij = lij / d;
            if (row) L[lane + j * D] = lij;
            fl += 1 + (nf - jpos - 1);
            ++jpos;
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
#pragma unroll
        for (int j = 0; j < D; ++j) {
            if (!in_mask(F, j)) continue;
            const double v = fabs(A[lane + j * D]);
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
        double s = b;
#pragma unroll 1
        for (int j = 0; j < D; ++j) {
            if (!in_mask(F, j)) continue;
            if (lane == j) s = s / ldiag;
            const double bj = bcast(s, j);
            if (in_mask(F, lane) && lane > j) s -= L[lane + j * D] * bj;
        }
        return s;
    }
    // dense.hpp:229-235 backward solve L^T b = rhs on F, exact order: for i
    // descending, s = b_i - sum_{j > i ascending} L(j,i) b_j.
    __device__ __forceinline__ double trsv_bwd(double b, unsigned F) {
        if (lane < D) buf[lane] = b;
        __syncwarp();
        double out = b;
#pragma unroll 1
        for (int i = D - 1; i >= 0; --i) {
            if (!in_mask(F, i)) continue;
            double s = buf[i];
#pragma unroll 1
            for (int j = i + 1; j < D; ++j)
                if (in_mask(F, j)) s -= L[j + i * D] * bb[j];
            const double bi = s / L[i + i * D];
            if (lane == i) {
                out = bi;
                bb[i] = bi;
            }
            __syncwarp();
        }
        __syncwarp();
        return out;
    }

    // ------------------------------------------------ tron.hpp:290-344
    // Steihaug PCG on the free set.  Returns 0 or an error status.
    // cg_status: 0 Converged, 1 Boundary, 2 NegCurve, 3 IterCap
    __device__ __forceinline__ int precond_cg(unsigned F, int nf, double gfree, double delta,
                                              double ldiag, double& step, int& cg_status,
                                              int& iters) {
        const long long nf2 = (long long)nf * nf;
        double w = 0.0;
        fl += nf;
        double bhat = trsv_fwd(gfree * -1.0, F, ldiag);
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
            if (sqrt(rtr) <= cfg.cg_tol * bnorm) {
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
    __device__ __forceinline__ double line_search(double x, double l, double u, double g, double w,
                                                  unsigned F) {
        const double kBetaFloor = 1e-12;
        double beta = 1.0;
        int bc;
        double bmin, bmax;
        breakpt(x, w, l, u, F, bc, bmin, bmax);
        bool search = true;
#pragma unroll 1
        while (search && beta > bmin && beta > kBetaFloor) {
            const double s = gpstep(x, beta, w, l, u, F);
            double gs;
            const double q = quad_model(g, s, F, gs);
            fl += 2 * __popc(F) + 1;
            if (q <= cfg.mu0 * gs) search = false;
            else beta *= cfg.interp_factor;
        }
        if (beta < 1.0 && beta < bmin) beta = bmin;
        fl += 2 * __popc(F);
        return clip(x + beta * w, l, u);
    }

    // tron.hpp:201-250.  Returns 0 or TB_STATUS_EVALUATION_ERROR.
    __device__ __forceinline__ int cauchy(double x, double g, double l, double u, double delta,
                                          double alpha_start, double& alpha_out, double& s) {
        const unsigned m = act;
        const int nn = n;
        const double radius = cfg.mu1 * delta;
        const double extrap_factor = 1.0 / cfg.interp_factor;
        double alpha = alpha_start;
        const double mg = -1.0 * g;
        fl += nn;
        int bc;
        double bmin, bmax;
        breakpt(x, mg, l, u, m, bc, bmin, bmax);
        s = gpstep(x, -alpha, g, l, u, m);
        bool interpolate;
        if (nrm2(s, m) > radius) {
            interpolate = true;
        } else {
            double gs;
            const double q = quad_model(g, s, m, gs);
            if (!isfinite(q)) return TB_STATUS_EVALUATION_ERROR;
            fl += 2 * nn + 1;
            interpolate = q >= cfg.mu0 * gs;
        }
        if (interpolate) {
            bool search = true;
#pragma unroll 1
            while (search && alpha > 1e-30) {
                alpha *= cfg.interp_factor;
                s = gpstep(x, -alpha, g, l, u, m);
                if (nrm2(s, m) <= radius) {
                    double gs;
                    const double q = quad_model(g, s, m, gs);
                    if (!isfinite(q)) return TB_STATUS_EVALUATION_ERROR;
                    fl += 2 * nn + 1;
                    search = q >= cfg.mu0 * gs;
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
                    if (q < cfg.mu0 * gs) alpha_good = alpha;
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
    __device__ __forceinline__ int subspace_step(double x0, double g, double l, double u,
                                                 double delta, double cs, double& xout,
                                                 double& sout, long long& cg_total) {
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
            if (sqrt(gfnormf) <= cfg.cg_tol * gfnorm) break;
            if (cgs == 1 || cgs == 3) break;
        }
        sout = s;
        return 0;
    }
};

// ------------------------------------------------------------ families
template <int FAM>
struct Family {
    // objective at the point staged in xs (all lanes, redundantly)
    static __device__ __forceinline__ double f(const double* xs, const double* prm, int n) {
        return tb_family_f(FAM, xs, prm, n);
    }
    static __device__ __forceinline__ double grad(const double* xs, const double* prm, int n, int i) {
        if (FAM == TB_FAMILY_HS45) return tb_hs45_grad_i(xs, n, i);
        if (FAM == TB_FAMILY_BOXQP) return tb_boxqp_grad_i(xs, prm, n, i);
        if (FAM == TB_FAMILY_NCVX) return tb_ncvx_grad_i(xs, prm, n, i);
        tb_branch_ctx c;
        tb_branch_ctx_init(xs, prm, n, &c);
        return tb_branch_grad_ctx(&c, i);
    }
    // row i of the Hessian into A[i + j*ld]
    static __device__ __forceinline__ void hess_row(const double* xs, const double* prm, int n, int i,
                                                    double* A, int ld) {
        if (FAM == TB_FAMILY_BRANCH) {
            tb_branch_ctx c;
            tb_branch_ctx_init(xs, prm, n, &c);
            for (int j = 0; j < n; ++j) A[i + j * ld] = tb_branch_hess_ctx(&c, prm, i, j);
            return;
        }
        for (int j = 0; j < n; ++j) {
            double v;
            if (FAM == TB_FAMILY_HS45) v = tb_hs45_hess(xs, n, i, j);
            else if (FAM == TB_FAMILY_BOXQP) v = tb_boxqp_hess(prm, n, i, j);
            else v = tb_ncvx_hess(xs, prm, n, i, j);
            A[i + j * ld] = v;
        }
    }
};

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

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <int D>
constexpr int smem_doubles_fixed() {
    return 2 * D * D + 3 * D;
}

// tron.hpp:453-549 solve(), one problem per warp (one warp per block).
template <int FAM, int D>
__global__ void __launch_bounds__(32) tron_solve_kernel(const KernelArgs a) {
    extern __shared__ double smem[];
    const long long pid = blockIdx.x;
    if (pid >= a.count) return;
    const unsigned long long t_start = globaltimer();

    Warp<D> W;
    W.A = smem;
    W.L = smem + D * D;
    W.buf = smem + 2 * D * D;
    W.bb = W.buf + D;
    W.xs = W.bb + D;
    double* prm_s = W.xs + D;
    W.n = a.n;
    W.lane = lane_id();
    W.act = (a.n >= 32) ? FULL : ((1u << a.n) - 1u);
    W.fl = 0;
    W.cfg = a.cfg;
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
    const double l = act ? a.lo[pid * n + lane] : 0.0;
    const double u = act ? a.up[pid * n + lane] : 0.0;
    double x = act ? a.x0[pid * n + lane] : 0.0;

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
        if (act) W.xs[lane] = x;
        __syncwarp();
        f = Family<FAM>::f(W.xs, prm_s, n);
        W.fl += tb_family_flops(FAM, n, 0);
        f_evals = 1;
        double g = act ? Family<FAM>::grad(W.xs, prm_s, n, lane) : 0.0;
        W.fl += tb_family_flops(FAM, n, 1);
        __syncwarp();
        pg = W.pgnorm(x, g, l, u);
        double delta = cfg.has_delta0 ? cfg.delta0 : tb_smax(W.nrm2(g, W.act), 1.0);
        double alpha_c = 1.0;
        bool need_hessian = true;
        status = pg <= cfg.tol_pg ? TB_STATUS_CONVERGED : TB_STATUS_ITER_LIMIT;

        if (status != TB_STATUS_CONVERGED) {
#pragma unroll 1
            for (int iter = 1; iter <= cfg.max_iter; ++iter) {
                iterations = iter;
                if (need_hessian) {
                    // x is staged in W.xs (at entry or after acceptance)
                    if (act) Family<FAM>::hess_row(W.xs, prm_s, n, lane, W.A, D);
                    W.fl += tb_family_flops(FAM, n, 2);
                    need_hessian = false;
                    __syncwarp();
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
                if (rc == TB_STATUS_FACTORIZATION_FAILED) {
                    status = TB_STATUS_FACTORIZATION_FAILED;
                    break;
                }
                if (rc) {
                    status = rc;
                    break;
                }
                cg_iterations += cg_its;
                // f at the trial point (stage it; restage x if rejected)
                if (act) W.xs[lane] = xt;
                __syncwarp();
                const double f_trial = Family<FAM>::f(W.xs, prm_s, n);
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
                    x = xt;  // W.xs already holds xt
                    f = f_trial;
                    g = act ? Family<FAM>::grad(W.xs, prm_s, n, lane) : 0.0;
                    W.fl += tb_family_flops(FAM, n, 1);
                    __syncwarp();
                    need_hessian = true;
                    pg = W.pgnorm(x, g, l, u);
                    if (pg <= cfg.tol_pg) {
                        status = TB_STATUS_CONVERGED;
                        break;
                    }
                } else {
                    if (act) W.xs[lane] = x;
                    __syncwarp();
                }
                if (delta <= 1e-300) break;
                // Zero-change fixed point: a rejected
                // iteration k >= 2 that leaves delta and alpha_c bitwise
                // unchanged leaves the whole solver state (x, f, g, A, delta,
                // alpha_c) unchanged, so every remaining iteration replays it
                // exactly.  Fast-forward with identical counters.
                if (a.fast_forward && !accepted && iter >= 2 && delta == delta_in &&
                    alpha_c == alpha_in) {
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
