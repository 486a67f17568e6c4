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

#ifndef TB_UNROLL_MAX
#define TB_UNROLL_MAX 6  // fully unroll the D-loops of kernels with D <= this (D = 8: masked loops,
                         // fewer live registers: ncvx8 6.09 -> 4.00 ms at 24 blocks/SM)
#endif
#ifndef TB_OUTLINE_SOLVES
#define TB_OUTLINE_SOLVES 0  // 1: one out-of-line copy of each triangular solve (measured slower)
#endif
#if TB_OUTLINE_SOLVES
#define TB_SOLVE_INLINE __noinline__
#else
#define TB_SOLVE_INLINE __forceinline__
#endif
#ifndef TB_MIN_BLOCKS
#define TB_MIN_BLOCKS 0  // > 0: force this many resident one-warp blocks per SM for every D
#endif

// Debug build only (-DTB_PHASES): per-phase clock64() accumulation, read back
// with tb_debug_read_phases() (scripts/phase_profile.py).
#ifdef TB_PHASES
#define TB_PH_BEGIN(k) const long long tb_ph_t0_##k = clock64();
#define TB_PH_END(w, k) (w).ph[k] += clock64() - tb_ph_t0_##k;
#else
#define TB_PH_BEGIN(k)
#define TB_PH_END(w, k)
#endif

namespace tbdev {

#ifdef TB_PHASES
__device__ unsigned long long g_phase_cycles[16];
#endif

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ bool in_mask(unsigned m, int i) { return (m >> i) & 1u; }
__device__ __forceinline__ int low_bit(unsigned m) { return __ffs(m) - 1; }
__device__ __forceinline__ int high_bit(unsigned m) { return 31 - __clz(m); }

// IEEE division kept out of line for rare paths (code size: the kernel's hot
// loop must stay small for the instruction cache).
static __device__ __noinline__ double div_ieee(double a, double d) { return a / d; }

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
    double extrap;  // 1.0 / cfg.interp_factor, computed on the host (IEEE, same bits)
    double* x_star;
    double* f_star;
    double* pg_norm;
    int32_t* status;
    int32_t* iterations;
    int64_t* cg_iterations;
    int64_t* f_evals;
    double* wall_time;
    int64_t* flops;
    // block kernel (d > 32) only: global workspace (work counter + per-block
    // Hessian slices) and its size in bytes
    void* ws;
    size_t ws_bytes;
    // problems of the whole batch / partition this launch is a chunk of
    // (kernel-form routing, tron_thread.cuh thread_form); 0 = count
    long long route_count;
    // persistent kernels (refilling thread form): problem counter, zeroed on
    // the launch stream before the launch
    unsigned long long* next;
    int form;  // TB_FORM_* requested by the context (routing only)
    // device flag: when non-null and set, the launch does nothing (ADMM
    // iterations enqueued past convergence, tb_admm_run)
    const int* skip;
    // launch order (tron_order.cu): the k-th block / thread / work item
    // solves problem order[k]; null = index order
    const uint32_t* order;
};



// shared memory per warp (doubles; every region starts at an even offset)
template <int D>
struct SmemLayout {
    static constexpr int GS = D <= 4 ? 4 : (D <= 8 ? 8 : (D <= 16 ? 16 : 32));
    static constexpr int A = 0;                      // D*D Hessian
    static constexpr int L = A + D * D;              // (32/GS)*D*D factors, one per lane group
    static constexpr int RD = L + (32 / GS) * D * D; // D reciprocal diagonal of the winning factor
    static constexpr int S1 = RD + D;                // 2*D ordered-sum staging (double buffered)
    static constexpr int S2 = S1 + 2 * D;    // 2*D second staging (double buffered)
    static constexpr int XS = S2 + 2 * D;    // D point for family evaluations
    static constexpr int CTX = XS + D;       // family context (branch: sizeof(tb_branch_ctx))
    static constexpr int CTX_DOUBLES = (int)((sizeof(tb_branch_ctx) / sizeof(double) + 1) & ~1);
    static constexpr int SC = CTX + CTX_DOUBLES;   // 8 warp-uniform loop scalars kept out of registers
    static constexpr int LU = SC + 8;              // bounds of lanes 0..31 (D = 8: Warp::kBoundsSmem)
    static constexpr int PRM = LU + (D == 8 ? 64 : 0);  // staged parameters
    static constexpr int fixed() { return PRM; }
    static_assert(D % 2 == 0, "D must be even (16-byte staging loads)");
};

#ifndef TB_FWD_REDUNDANT
#define TB_FWD_REDUNDANT 0
#endif

// ------------------------------------------------------------ solves
// Correctly rounded a / d from r = RN(1/d) (Markstein): q0 = RN(a r),
// e = a - d q0 exactly (FMA), RN(q0 + e r) == RN(a / d) when no intermediate
// is subnormal / huge; zero, subnormal, huge, inf and NaN quotients take the
// IEEE division.  3 dependent ops instead of ~15 (DDIV ~125 cycles).
__device__ __forceinline__ double div_rcp(double a, double d, double r) {
    const double q0 = a * r;
    const unsigned ex = ((unsigned)__double2hiint(q0) >> 20) & 0x7FFu;
    if (ex - 64u > 1918u) return div_ieee(a, d);
    const double e = fma(-q0, d, a);
    return fma(e, r, q0);
}

// The same quotient without the branch: the range test only sets `bad`.  A
// branch on a value computed from the quotient stalls the warp until the
// test resolves (~100 cycles per quotient in a dependent chain, measured:
// scripts/micro/latency.cu), so the triangular solves run every quotient
// through this form and test `bad` once at the end; a solve that met an
// out-of-range quotient is recomputed with IEEE divisions (identical results
// to div_rcp everywhere).
template <bool IEEE>
__device__ __forceinline__ double quot(double a, double d, double r, bool& bad) {
    if (IEEE) return a / d;
    const double q0 = a * r;
    const unsigned ex = ((unsigned)__double2hiint(q0) >> 20) & 0x7FFu;
    bad |= ex - 64u > 1918u;
    const double e = fma(-q0, d, a);
    return fma(e, r, q0);
}

// dense.hpp:224-228 forward solve L b = rhs on F (column sweep == the
// reference's ascending row dot-form, element by element); lane j's value is
// broadcast and every lane divides it (uniform operands, no divergence).
// Fully unrolled builds run the row dot-form redundantly on every lane instead
// (the right-hand side gathered once up front; identical bits on all lanes).
template <int D, bool UNROLL, bool IEEE>
__device__ __forceinline__ double trsv_fwd_core(const double* __restrict__ Lw, const double* __restrict__ RD, double b,
                                                unsigned F, int lane, bool& bad) {
    const bool inF = lane < D && in_mask(F, lane);
#if TB_FWD_REDUNDANT
    if (UNROLL) {
        double bv[D];
#pragma unroll
        for (int j = 0; j < D; ++j) bv[j] = __shfl_sync(FULL, b, j);
        double out = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            if (!in_mask(F, i)) continue;
            double s = bv[i];
#pragma unroll
            for (int j = 0; j < i; ++j)
                if (in_mask(F, j)) s -= Lw[i + j * D] * bv[j];
            bv[i] = quot<IEEE>(s, Lw[i + i * D], RD[i], bad);
            if (lane == i) out = bv[i];
        }
        return out;
    }
#endif
    double s = inF ? b : 0.0;
    auto step = [&](int j) {
        const double q = quot<IEEE>(__shfl_sync(FULL, s, j), Lw[j + j * D], RD[j], bad);
        if (lane == j) s = q;
        else if (inF && lane > j) s -= Lw[lane + j * D] * q;
    };
    if (UNROLL) {
#pragma unroll
        for (int j = 0; j < D; ++j)
            if (in_mask(F, j)) step(j);
    } else {
#pragma unroll 1
        for (unsigned mj = F; mj; mj &= mj - 1) step(low_bit(mj));
    }
    return s;
}

// dense.hpp:229-235 backward solve L^T b = rhs on F, exact order: for i
// descending, s = b_i - sum_{j > i ascending} L(j,i) b_j.  Every lane computes
// every b_i (redundantly, identical bits); bb is D doubles of staging.
template <int D, bool UNROLL, bool IEEE>
__device__ __forceinline__ double trsv_bwd_core(const double* __restrict__ Lw, const double* __restrict__ RD,
                                                double* __restrict__ bb, double b, unsigned F, int lane, bool& bad) {
    double out = b;
    if (UNROLL) {
        double bv[D];
#pragma unroll
        for (int i = D - 1; i >= 0; --i) {
            bv[i] = 0.0;
            if (!in_mask(F, i)) continue;
            double s = __shfl_sync(FULL, b, i);
#pragma unroll
            for (int j = i + 1; j < D; ++j)
                if (in_mask(F, j)) s -= Lw[j + i * D] * bv[j];
            bv[i] = quot<IEEE>(s, Lw[i + i * D], RD[i], bad);
            if (lane == i) out = bv[i];
        }
    } else {
#pragma unroll 1
        for (unsigned mi = F; mi; mi &= ~(1u << high_bit(mi))) {
            const int i = high_bit(mi);
            double s = __shfl_sync(FULL, b, i);
#pragma unroll 1
            for (unsigned mj = F & ~((2u << i) - 1u); mj; mj &= mj - 1) {
                const int j = low_bit(mj);
                s -= Lw[j + i * D] * bb[j];
            }
            const double bi = quot<IEEE>(s, Lw[i + i * D], RD[i], bad);
            if (lane == i) {
                out = bi;
                bb[i] = bi;
            }
            __syncwarp();
        }
    }
    return out;
}

// the rare recomputation with IEEE divisions, out of line
template <int D, bool UNROLL>
__device__ __noinline__ double trsv_fwd_ieee(const double* Lw, const double* RD, double b, unsigned F, int lane) {
    bool bad = false;
    return trsv_fwd_core<D, UNROLL, true>(Lw, RD, b, F, lane, bad);
}
template <int D, bool UNROLL>
__device__ __noinline__ double trsv_bwd_ieee(const double* Lw, const double* RD, double* bb, double b, unsigned F,
                                             int lane) {
    bool bad = false;
    return trsv_bwd_core<D, UNROLL, true>(Lw, RD, bb, b, F, lane, bad);
}

// `bad` is warp-uniform: every lane forms every quotient from the same operands
template <int D, bool UNROLL>
__device__ TB_SOLVE_INLINE double trsv_fwd_fn(const double* __restrict__ Lw, const double* __restrict__ RD, double b,
                                             unsigned F, int lane) {
    bool bad = false;
    const double out = trsv_fwd_core<D, UNROLL, false>(Lw, RD, b, F, lane, bad);
    return bad ? trsv_fwd_ieee<D, UNROLL>(Lw, RD, b, F, lane) : out;
}
template <int D, bool UNROLL>
__device__ TB_SOLVE_INLINE double trsv_bwd_fn(const double* __restrict__ Lw, const double* __restrict__ RD,
                                             double* __restrict__ bb, double b, unsigned F, int lane) {
    bool bad = false;
    const double out = trsv_bwd_core<D, UNROLL, false>(Lw, RD, bb, b, F, lane, bad);
    return bad ? trsv_bwd_ieee<D, UNROLL>(Lw, RD, bb, b, F, lane) : out;
}

// ---------------------------------------------------------------- per warp
template <int D, bool COUNT>
struct Warp {
    static constexpr bool kUnroll = D <= TB_UNROLL_MAX;
    double* A;
    double* L;   // G*D*D: one factor per lane group (parallel shift attempts)
    double* Lw;  // the successful attempt's factor
    double* RD;  // D: RN(1 / L(i,i)) of Lw
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
    // factor memo (ccf): the free set of the last successful factorization of
    // the current Hessian, and its flops (COUNT builds)
    unsigned memo_F;
    bool memo_ok;
    long long memo_fl;
    bool memo_credit;  // credit a memoised call's flops (fast_forward 1: the reference's count; 2: executed only)
    double extrap;  // 1.0 / cfg->interp_factor
    // D = 8 keeps the bounds in shared memory (l at lu[lane], u at lu[32 + lane])
    // and re-reads them where used, so they are not live across ccf / PCG:
    // fewer spills in the masked-loop kernel (ncvx8 x32,768 3.39 -> 3.14 ms;
    // the other D measured 2-4 % slower that way and keep registers;
    // profiles/r02_ab_bounds_smem.txt)
    static constexpr bool kBoundsSmem = D == 8;
    // this lane's bounds: the shared-memory slots (D = 8, read here) or the
    // register value the caller holds
    __device__ __forceinline__ double lb(double l) const {
        if constexpr (kBoundsSmem)
            return static_cast<const volatile double*>(s1 + (SmemLayout<D>::LU - SmemLayout<D>::S1))[lane];
        else
            return l;
    }
    __device__ __forceinline__ double ub(double u) const {
        if constexpr (kBoundsSmem)
            return static_cast<const volatile double*>(s1 + (SmemLayout<D>::LU - SmemLayout<D>::S1))[32 + lane];
        else
            return u;
    }
#ifdef TB_PHASES
    long long ph[8];
#endif

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
    // Shift escalation in parallel (dense.hpp:182-201).  The reference tries
    // A + a_k I for a_0 = 0, a_{k+1} = max(2 a_k, alpha0), k = 0, 1, ...
    // sequentially until one factorization succeeds (cap -> failure).  Every
    // attempt is an independent function of (A[F,F], a_k), so G lane groups of
    // GS >= D lanes each run attempts k0 .. k0+G-1 at once; the first success
    // in k order is the reference's result (same L, same shift, same flop
    // count).  Within a group, lane i owns row i of the current column
    // (left-looking, dense.hpp:141-154: zero-skip on L(j,k), pivot test
    // !(pivot > 0), division by sqrt(pivot)).
    static constexpr int GS = D <= 4 ? 4 : (D <= 8 ? 8 : (D <= 16 ? 16 : 32));
    static constexpr int G = 32 / GS;

    // one round of G attempts; returns the winning group or -1.  `fl_round`
    // receives the flops the reference spends on the attempts up to and
    // including the winner (all G if none wins).
    __device__ __forceinline__ int chol_round(unsigned F, int nf, double sh, bool valid, long long& fl_round) {
        const int g = lane / GS, i = lane % GS;
        double* Lg = L + g * D * D;
        const bool inF = i < D && in_mask(F, i);
        bool alive = valid;
        int rem = nf;
        int my_fl = 0;  // flops of this group's attempt (counted on lane i == 0)
        auto column = [&](int j) {
            const bool row = alive && inF && i >= j;
            double lij = row ? A[i + j * D] : 0.0;
            if (i == j) lij += sh;
            int cnt = 0;
            auto kstep = [&](int k) {
                const double ljk = Lg[j + k * D];
                const bool nz = ljk != 0.0;
                if (nz && row) lij -= ljk * Lg[i + k * D];
                cnt += nz;
            };
            if (kUnroll) {
#pragma unroll
                for (int k = 0; k < D - 1; ++k)
                    if (k < j && in_mask(F, k)) kstep(k);
            } else {
#pragma unroll 1
                for (unsigned mk = F & ((1u << j) - 1u); mk; mk &= mk - 1) kstep(low_bit(mk));
            }
            const double pivot = __shfl_sync(FULL, lij, j, GS);
            const bool ok = pivot > 0.0;
            if (alive) my_fl += 1 + 2 * rem * cnt + (ok ? rem : 0);
            const double d = sqrt(ok ? pivot : 1.0);
            const double q = lij / d;
            if (row && ok) Lg[i + j * D] = i == j ? d : q;
            alive = alive && ok;
            --rem;
            __syncwarp();
        };
        // Unrolled (D <= 6): every column of F, without a per-column vote on
        // the groups' pivots -- a vote + branch in the column chain costs more
        // than the columns a round whose attempts all fail early would skip
        // (dead groups neither store nor count).  Masked loops (D >= 8, where
        // failing rounds are long) stop once every group has failed.
        if (kUnroll) {
#pragma unroll
            for (int j = 0; j < D; ++j)
                if (in_mask(F, j)) column(j);
        } else {
#pragma unroll 1
            for (unsigned mj = F; mj && __any_sync(FULL, alive); mj &= mj - 1) column(low_bit(mj));
        }
        const unsigned wins = __ballot_sync(FULL, i == 0 && alive);
        const int winner = wins ? low_bit(wins) / GS : -1;
        if (COUNT) {
            const int last = winner >= 0 ? winner : G - 1;
            // failed attempts also pay the alpha update (dense.hpp:197)
            const int contrib = (i == 0 && valid && g <= last) ? my_fl + (g < winner || winner < 0 ? 1 : 0) : 0;
            fl_round = __reduce_add_sync(FULL, (unsigned)contrib);
        }
        return winner;
    }

#ifndef TB_CCF_MEMO
#define TB_CCF_MEMO 1
#endif
    // Factor memo: ccf is a pure function of A[F,F].  While the Hessian is
    // unchanged (rejected steps; hess() clears memo_ok) and the free set
    // repeats -- the stagnating tail of a solve, repeated faces -- the factor
    // Lw / RD left by the previous call is the reference's result again (its
    // shift attempts would replay identically, same flops), so it is reused.
    // The factor region is written by ccf alone, so Lw / RD are intact.
    __device__ __forceinline__ int ccf(unsigned F, int nf) {
        if (TB_CCF_MEMO && memo_ok && F == memo_F) {
            if (memo_credit) count(memo_fl);
            return 0;
        }
        const long long fl0 = fl;
        double shift;
        const int rc = ccf_compute(F, nf, shift);
        memo_ok = TB_CCF_MEMO && rc == 0;
        memo_F = F;
        if (COUNT) memo_fl = fl - fl0;
        return rc;
    }

    // dense.hpp:182-201 shifted_factorize on A[F,F].  On success Lw points at
    // the factor and RD holds RN(1 / L(i,i)).  Returns 0 or
    // TB_STATUS_FACTORIZATION_FAILED.
    __device__ __forceinline__ int ccf_compute(unsigned F, int nf, double& shift) {
        const bool inF = lane < D && in_mask(F, lane);
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
        const int g = lane / GS;
        double base = 0.0;  // a_{k0}
#pragma unroll 1
        for (int k0 = 0; k0 < 4096; k0 += G) {
            // a_{k0+g}: closed form (tb_math.h); at G = 2 the single step
            // (D = 16: the closed form measured 1.6 % slower there)
            const double sh = G <= 2 ? (g ? tb_smax(2.0 * base, alpha0) : base) : tb_shift_ahead(base, alpha0, g);
            const bool valid = (k0 + g == 0) || (sh <= cap);
            long long flr = 0;
            const int w = chol_round(F, nf, sh, valid, flr);
            count(flr);
            if (w >= 0) {
                shift = __shfl_sync(FULL, sh, w * GS);
                Lw = L + w * D * D;
                if (lane < D) {
                    const double dii = Lw[lane + lane * D];
                    RD[lane] = inF ? __drcp_rn(dii) : 1.0;  // RN(1/d): the bits of 1.0 / d
                }
                __syncwarp();
                return 0;
            }
            // no success among attempts k0..k0+G-1: the reference throws at
            // the first a_k > cap (all earlier attempts failed)
            if (!__all_sync(FULL, valid)) return TB_STATUS_FACTORIZATION_FAILED;
            if (G <= 2) {
                for (int t = 0; t < G; ++t) base = tb_smax(2.0 * base, alpha0);
            } else {
                base = tb_shift_ahead(base, alpha0, G);
            }
        }
        // unreachable for finite data (alpha doubles past any finite cap);
        // with an infinite cap the reference never terminates
        return TB_STATUS_FACTORIZATION_FAILED;
    }

    __device__ __forceinline__ double trsv_fwd(double b, unsigned F, double, double) {
        return trsv_fwd_fn<D, kUnroll>(Lw, RD, b, F, lane);
    }
    __device__ __forceinline__ double trsv_bwd(double b, unsigned F) {
        // staging for the non-unrolled variant only: the unrolled one neither
        // stages nor synchronises, so it must not advance the staging toggle
        // (a toggle without a barrier would let the next staged write reuse a
        // buffer other lanes may still read: racecheck, r02_sanitize_racecheck)
        double* bb = s2 + tog;
        if (!kUnroll) tog ^= D;
        return trsv_bwd_fn<D, kUnroll>(Lw, RD, bb, b, F, lane);
    }

    // ------------------------------------------------ tron.hpp:290-344
    // Steihaug PCG on the free set.  Returns 0 or an error status.
    // cg_status: 0 Converged, 1 Boundary, 2 NegCurve, 3 IterCap
    __device__ __forceinline__ int precond_cg(unsigned F, int nf, double gfree, double delta, double ldiag,
                                              double rdiag, double& step, int& cg_status, int& iters) {
        const long long nf2 = (long long)nf * nf;
        double w = 0.0;
        count(nf);
        const double bhat = trsv_fwd(gfree * -1.0, F, ldiag, rdiag);
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
            q = trsv_fwd(q, F, ldiag, rdiag);
            count(2 * nf2);
            const double ptq = dot(p, q, F);
            // both branches of tron.hpp:315-327 call trqsol(w, p, delta) on
            // the same inputs: one call site (code size), same result / error
            double sigma;
            const int rc = trqsol(w, p, delta, F, sigma);
            if (rc) return rc;
            if (ptq <= 0.0) {
                w += sigma * p;
                count(2 * nf);
                cg_status = 2;
                break;
            }
            const double alpha = rho / ptq;
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
        const double extrap_factor = extrap;  // 1.0 / interp_factor (tron.hpp:204), once per solve
        double alpha = alpha_start;
        const double mg = -1.0 * g;
        count(nn);
        double bmin, bmax;
        breakpt(x, mg, l, u, m, bmin, bmax);
        // The reference's initial test, interpolation loop and extrapolation
        // loop (tron.hpp:210-248) as one state machine with a single trial
        // site (code size): same trials in the same order, same flops.
        int mode = 0;  // 0 initial test, 1 interpolate, 2 extrapolate
        double alpha_good = alpha;
#pragma unroll 1
        for (;;) {
            s = gpstep(x, -alpha, g, l, u, m);
            const double nr = nrm2(s, m);
            // :212 evaluates q unless nrm > radius; :224/:235 only if nrm <= radius
            const bool evalq = mode == 0 ? !(nr > radius) : (nr <= radius);
            bool qge = false;  // q >= mu0 g's (q and g's are finite here)
            if (evalq) {
                double gs;
                const double q = quad_model(g, s, m, gs);
                if (!isfinite(q)) return TB_STATUS_EVALUATION_ERROR;
                count(2 * nn + 1);
                qge = q >= cfg->mu0 * gs;
            }
            if (mode == 0) {
                if (!evalq || qge) {  // interpolate
                    mode = 1;
                    if (!(alpha > 1e-30)) break;
                    alpha *= cfg->interp_factor;
                    continue;
                }
                mode = 2;  // extrapolate
                alpha_good = alpha;
                if (!(alpha <= bmax)) break;
                alpha *= extrap_factor;
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
                alpha *= extrap_factor;
                continue;
            }
            break;
        }
        if (mode == 2) {
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
#define TB_LB lb(l)
#define TB_UB ub(u)
        xout = clip(x0 + 1.0 * cs, TB_LB, TB_UB);
        count(2 * nn);
        double s = xout - x0;
        count(nn);
        double w = gemv(s, act);
        cg_total = 0;
#pragma unroll 1
        for (int faces = 0; faces < nn; ++faces) {
            const bool fr = lane < nn && TB_LB < xout && xout < TB_UB;
            const unsigned F = __ballot_sync(FULL, fr);
            const int nf = __popc(F);
            if (nf == 0) break;
            TB_PH_BEGIN(2)
            int rc = ccf(F, nf);
            TB_PH_END(*this, 2)
            if (rc) return rc;
            const double ldiag = fr ? Lw[lane + lane * D] : 1.0;
            const double rdiag = fr ? RD[lane] : 1.0;
            if (__any_sync(FULL, fr && ldiag == 0.0)) return TB_STATUS_SINGULAR_FACTOR;
            const double gfree = w + g;
            count(nf);
            const double gfnorm = nrm2(g, F);
            double step;
            int cgs, its;
            TB_PH_BEGIN(3)
            rc = precond_cg(F, nf, gfree, delta, ldiag, rdiag, step, cgs, its);
            TB_PH_END(*this, 3)
            if (rc) return rc;
            cg_total += its;
            TB_PH_BEGIN(4)
            const double xn = line_search(xout, TB_LB, TB_UB, gfree, step, F);
            TB_PH_END(*this, 4)
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
#undef TB_LB
#undef TB_UB
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

    // the solver's family interface (tron_solve_one): the per-point context
    // region in shared memory, and the flop model of the evaluations
    __device__ __forceinline__ void bind(double* context) { ctx = reinterpret_cast<tb_branch_ctx*>(context); }
    __device__ __forceinline__ static long long flops(int n, int kind) { return tb_family_flops(FAM, n, kind); }

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
            }
        }
        if (FAM == TB_FAMILY_BRANCH) {
            // one lower-triangle entry per lane (n(n+1)/2 <= 21 entries);
            // tb_br_hess canonicalises (i, j) so both halves get the same bits
            int a = 0, b = lane;
            while (b > a) {
                b -= a + 1;
                ++a;
            }
            if (a < n) {
                const double h = tb_br_hess(ctx, prm, n, a, b);
                W.A[a + b * D] = h;
                W.A[b + a * D] = h;
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

// Resident one-warp blocks per SM the register budget targets (the kernel is
// latency-bound and its SM throughput grows with resident warps; a few
// spilled registers cost less than the lost residency).  Measured on B200,
// device-resident batches: D=6 C2 9.56 / 8.89 / 8.43 / 8.28 /
// 9.14 ms at 16 / 18 / 22 / 24 / 28 before the loop scalars moved to shared
// memory, 8.22 / 8.09 ms at 24 / 28 after; after the register diet D=4 and
// D=8 (masked loops) also run best at 28 (ncvx4 1.537 -> 1.495 ms, branch4
// 1.363 -> 1.334, ncvx8 3.82 -> 3.69); D=16 at 20, 32 blocks always slower.
template <int D>
struct WarpMinBlocks {
    static constexpr int value = TB_MIN_BLOCKS > 0 ? TB_MIN_BLOCKS
                                 : D <= 8          ? 28
                                 : D <= 16         ? 20
                                                   : 16;
};

// tron.hpp:453-549 solve() of problem `pid` by one warp (the calling warp owns
// `smem`, SmemLayout<D>::fixed() + params doubles).
// FamT: the family's device evaluation (DevFamily for the built-in families;
// include/tronbatch_gpu/user_family.cuh wraps a caller's own type) with
// bind / prepare / f / grad / hess / flops.
template <int FAM, int D, bool COUNT, class FamT = DevFamily<FAM, D, COUNT>>
__device__ __forceinline__ void tron_solve_one(const KernelArgs& a, const long long pid, double* smem) {
    using SL = SmemLayout<D>;
    const unsigned long long t_start = globaltimer();

    Warp<D, COUNT> W;
    W.A = smem + SL::A;
    W.L = smem + SL::L;
    W.Lw = W.L;
    W.RD = smem + SL::RD;
    W.s1 = smem + SL::S1;
    W.s2 = smem + SL::S2;
    W.xs = smem + SL::XS;
    double* prm_s = smem + SL::PRM;
    W.n = a.n;
    W.lane = lane_id();
    W.tog = 0;
    W.act = (a.n >= 32) ? FULL : ((1u << a.n) - 1u);
    W.fl = 0;
    W.memo_F = 0;
    W.memo_ok = false;
    W.memo_fl = 0;
    W.memo_credit = a.fast_forward != 2;
#ifdef TB_PHASES
    for (int k = 0; k < 8; ++k) W.ph[k] = 0;
    const long long tb_ph_total0 = clock64();
#endif
    W.cfg = &a.cfg;
    W.extrap = a.extrap;
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
    FamT fam;
    fam.bind(smem + SL::CTX);
    constexpr bool kBS = Warp<D, COUNT>::kBoundsSmem;
    if constexpr (kBS) {
        volatile double* lus = smem + SL::LU;
        lus[lane] = act ? a.lo[pid * n + lane] : 0.0;
        lus[32 + lane] = act ? a.up[pid * n + lane] : 0.0;
    }
    const double l = kBS ? 0.0 : (act ? a.lo[pid * n + lane] : 0.0);
    const double u = kBS ? 0.0 : (act ? a.up[pid * n + lane] : 0.0);
#define TB_L W.lb(l)
#define TB_U W.ub(u)
    double x = act ? a.x0[pid * n + lane] : 0.0;
    __syncwarp();

    // warp-uniform loop state in shared memory (registers are the residency
    // limit, §4a).  The counters (read-modify-write) are updated and read by
    // lane 0 alone.  The other slots take warp-uniform values that every lane
    // stores identically; f, delta_in and alpha_in, which every lane reads
    // before they are rewritten in the same pass, are rewritten only after a
    // __syncwarp, so no lane can overwrite a value another lane has yet to
    // read (independent thread scheduling).
    double* sc = smem + SL::SC;
    double& delta_in = sc[0];  // delta / alpha_c at the start of the iteration (zero-change check)
    double& alpha_in = sc[1];
    long long& cg_iterations = reinterpret_cast<long long*>(sc)[2];
    long long& f_evals = reinterpret_cast<long long*>(sc)[3];
    double& f = sc[4];
    double& pg = sc[5];
    int& iterations = reinterpret_cast<int*>(sc + 6)[0];
    int& status = reinterpret_cast<int*>(sc + 6)[1];
    status = TB_STATUS_ITER_LIMIT;
    iterations = 0;
    cg_iterations = 0;
    f_evals = 0;
    f = 0.0;
    pg = 0.0;

    // tron.hpp:465-466
    if (__any_sync(FULL, act && !(TB_L <= TB_U))) {
        status = TB_STATUS_INVALID_BOUNDS;
    } else {
        const double kEta1 = 0.25, kEta2 = 0.75;
        // tron.hpp:473-549 restructured around ONE family-evaluation site and
        // ONE gradient site (code size: the branch context is large): pass 0
        // evaluates the start point (:473-483), pass k >= 1 the trial point of
        // iteration k (:506-539).  Same operations in the same order.
        x = W.clip(x, TB_L, TB_U);
        double xe = x;  // point being evaluated
        double g = 0.0, s = 0.0, delta = 0.0, alpha_c = 1.0;
        bool need_hessian = true;
        long long fl_iter0 = 0, cg_its = 0;
        delta_in = 0.0;
        alpha_in = 0.0;
#pragma unroll 1
        for (int iter = 0;; ++iter) {
            TB_PH_BEGIN(6)
            fam.prepare(W, xe);
            const double fe = fam.f(W);
            W.count(FamT::flops(n, 0));
            if (lane == 0) ++f_evals;
            TB_PH_END(W, 6)
            bool take = iter == 0;  // evaluate the gradient at xe
            if (iter > 0) {
                const double f_trial = fe;
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
                take = actred > cfg.eta0 * prered;  // accepted (:529)
                if (take) {
                    x = xe;
                    __syncwarp();  // every lane has read f (actred, alphax)
                    f = f_trial;
                    need_hessian = true;
                }
            } else {
                f = fe;
            }
            if (take) {
                g = fam.grad(W);  // the context was prepared at xe
                W.count(FamT::flops(n, 1));
                pg = W.pgnorm(x, g, TB_L, TB_U);
            }
            if (iter == 0) {
                delta = cfg.has_delta0 ? cfg.delta0 : tb_smax(W.nrm2(g, W.act), 1.0);
                status = pg <= cfg.tol_pg ? TB_STATUS_CONVERGED : TB_STATUS_ITER_LIMIT;
                if (status == TB_STATUS_CONVERGED) break;
            } else {
                if (take && pg <= cfg.tol_pg) {
                    status = TB_STATUS_CONVERGED;
                    break;
                }
                if (delta <= 1e-300) break;
                // Zero-change fixed point: a rejected
                // iteration k >= 2 that leaves delta and alpha_c bitwise
                // unchanged leaves the whole solver state (x, f, g, A, delta,
                // alpha_c) unchanged, so every remaining iteration replays it
                // exactly.  Fast-forward with identical counters.
                if (a.fast_forward && !take && iter >= 2 && delta == delta_in && alpha_c == alpha_in) {
                    const long long rem = cfg.max_iter - iter;
                    if (lane == 0) {
                        cg_iterations += rem * cg_its;
                        f_evals += rem;
                    }
                    if (a.fast_forward == 1) W.count(rem * (W.fl - fl_iter0));  // 2: executed flops only
                    iterations = cfg.max_iter;
                    break;
                }
            }
            if (iter + 1 > cfg.max_iter) break;
            iterations = iter + 1;
            if (need_hessian) {  // family context holds the current x
                TB_PH_BEGIN(0)
                fam.hess(W);
                TB_PH_END(W, 0)
                W.count(FamT::flops(n, 2));
                need_hessian = false;
                W.memo_ok = false;  // a new Hessian: the memoised factor is stale
            }
            fl_iter0 = W.fl;
            __syncwarp();  // every lane has read delta_in / alpha_in (zero-change test)
            delta_in = delta;
            alpha_in = alpha_c;

            double cs, alpha_new;
            TB_PH_BEGIN(1)
            int rc = W.cauchy(x, g, TB_L, TB_U, delta, alpha_c, alpha_new, cs);
            TB_PH_END(W, 1)
            if (rc) {
                status = rc;
                break;
            }
            alpha_c = alpha_new;
            TB_PH_BEGIN(5)
            rc = W.subspace_step(x, g, l, u, delta, cs, xe, s, cg_its);
            TB_PH_END(W, 5)
            if (rc) {
                status = rc;  // FactorizationFailed caught like tron.hpp:499-501
                break;
            }
            if (lane == 0) cg_iterations += cg_its;
        }
    }

#ifdef TB_PHASES
    W.ph[7] = clock64() - tb_ph_total0;
    if (lane == 0)
        for (int k = 0; k < 8; ++k) atomicAdd(&g_phase_cycles[k], (unsigned long long)W.ph[k]);
#endif
    __syncwarp();  // every lane's last store of the loop scalars before lane 0 reports them
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
#undef TB_L
#undef TB_U
}

// Small batches (at most kLatencyBlocks one-warp blocks per SM) are latency-
// bound: every problem is resident at once, so registers beyond the
// throughput variant's budget cost nothing and remove the spills (128 vs 72
// registers at D = 4 / 6 / 8): C1 ncvx4 x1,024 0.306 -> 0.277 ms, ncvx8
// x1,024 1.264 -> 1.158, branch6 x2,048 2.234 -> 2.071 (profiles/README.md).
constexpr int kLatencyBlocks = 16;

// One problem per warp (one warp per block); MINB resident blocks per SM.
// ORD: launch slot k solves problem a.order[k] (tron_order.cu; a separate
// instantiation, so index-order launches keep their code unchanged).
template <int FAM, int D, bool COUNT, int MINB = WarpMinBlocks<D>::value, bool ORD = false>
__global__ void __launch_bounds__(32, MINB) tron_solve_kernel(const __grid_constant__ KernelArgs a) {
    extern __shared__ double smem[];
    const long long pid = blockIdx.x;
    if (pid >= a.count || (a.skip && *a.skip)) return;
    tron_solve_one<FAM, D, COUNT>(a, ORD ? (long long)a.order[pid] : pid, smem);
}

}  // namespace tbdev
