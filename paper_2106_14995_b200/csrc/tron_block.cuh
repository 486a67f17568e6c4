// tron_block.cuh — one thread block solves one bound-constrained problem,
// 32 < d <= 128 (BASELINE config C3: the dimension sweep up to d = 128).
//
// The warp kernel (tron_device.cuh) keeps every vector in one register per
// lane and the Hessian plus up to 8 factor attempts in shared memory; past
// d = 32 that no longer fits a warp, so this variant uses D = 64 or 128
// threads (thread t owns variable t) and is organised around the shared-memory
// budget, which sets how many problems an SM holds:
//
//  * The free-set systems are COMPACTED, exactly like the reference
//    (tron.hpp:405-412 builds B = A[F,F]): each face pass ranks the free
//    variables, and the factor L of B is stored packed lower-triangular,
//    column-major, with leading dimension nf (nf(nf+1)/2 doubles, 66 KB at
//    nf = 128).  The preconditioned CG runs in compacted coordinates (thread
//    p owns the p-th free variable), so every loop is the reference's dense
//    loop over 0..nf-1 in the same order.
//  * The Hessian A (D x D) lives either in shared memory (ASMEM) or in a
//    per-resident-block slice of a global workspace that stays L2-resident;
//    the kernel is persistent (grid = SMs x resident blocks, problems taken
//    from an atomic work counter), so the workspace is sized by the grid,
//    not the batch, and long-running problems do not leave SMs idle.
//  * Parameters are read from global memory (ncvx at d = 128 carries 69 KB).
//
// Exactness is the same contract as the warp kernel (nvcc --fmad=false,
// ordered ascending sums, IEEE sqrt / division, std::min/max semantics):
//  * ordered sums are staged by ascending rank and summed serially over the
//    rank range (dense.hpp:81-83 over the compacted vector);
//  * Cholesky is left-looking per element (dense.hpp:141-154): thread p owns
//    row p of the current column, k ascending, zero-skip on L(j,k), division
//    by sqrt(pivot).  The normalisation L(p,j) = raw / d of a column is done
//    lazily at the start of the next column so one barrier per column
//    suffices; the value is the same IEEE quotient;
//  * the forward solve is a column sweep (element order == the reference's
//    row dot-form), the backward solve runs serially in ascending j per
//    element (dense.hpp:230-234) on warp 0.
#pragma once

#include "tron_device.cuh"

#ifndef TB_HESS_CONST_PART
#define TB_HESS_CONST_PART 1  // keep the x-independent Hessian part across evaluations (block kernel)
#endif
#ifndef TB_BLK_MIN128
#define TB_BLK_MIN128 4  // resident D = 128 blocks per SM (registers / shared factor region)
#endif
#ifndef TB_BLK_MIN32
#define TB_BLK_MIN32 16  // D = 32: one warp per problem
#endif
#ifndef TB_BLK_MIN64
#define TB_BLK_MIN64 8
#endif

namespace tbdev {

template <int D, bool ASMEM>
struct BlkLayout {
    static constexpr int NW = D / 32;
    // shared factor region: every packed factor for nf <= D at D = 64; at
    // D = 128 sized for 4 resident blocks per SM (2 parallel attempts at
    // nf <= 64, one factor up to nf = 108); larger systems use the block's
    // global fallback slice (LPFULL doubles)
    static constexpr int LPFULL = D * (D + 1) / 2;
    static constexpr int LP = D >= 128 ? (TB_BLK_MIN128 >= 5 ? 4352 : 5840) : LPFULL;
    static constexpr int L = 0;
    static constexpr int RD = L + LP;                // RN(1 / L(p,p))
    static constexpr int SW = 2 * D < 128 ? 128 : 2 * D;  // staging width (warp PCG uses 128)
    static constexpr int S1 = RD + D;                // staging, double buffered
    static constexpr int S2 = S1 + SW;
    static constexpr int S3 = S2 + SW;
    static constexpr int BB = S3 + SW;               // triangular-solve results
    static constexpr int XS = BB + D;                // evaluation point
    static constexpr int MISC = XS + D;              // 104 doubles of scalars (BM_*)
    static constexpr int FIDX = MISC + 104;          // D int32: free index by rank
    static constexpr int MSK = FIDX + D / 2;         // 2 x NW uint32 ballot words
    static constexpr int AS = MSK + ((NW + 1) & ~1); // Hessian (ASMEM only)
    static constexpr int total() { return AS + (ASMEM ? D * D : 0); }
    static_assert(LP % 2 == 0, "alignment");
};
// MISC slots
// BM_MEMO: ccf memo -- [0] flag (int), [1] flops (long long), [2..3] free-set ballot words (NW <= 4 uint32)
enum { BM_RED = 0, BM_PID = 16, BM_GOK = 18, BM_GFL = 22, BM_GRP = 30, BM_PCG = 62, BM_SC = 64, BM_MEMO = 96,
       BM_MISC_SIZE = 104 };

// a subset of the variables: its size and this thread's ascending rank in it
// (-1 if absent).  The staged vector of a subset is indexed by rank.
struct BSet {
    int cnt;
    int pos;
};

template <int D, bool ASMEM, bool COUNT>
struct Blk {
    using SL = BlkLayout<D, ASMEM>;
    static constexpr int NW = SL::NW;
    double* A;       // D x D column-major (shared or global workspace)
    double* L;       // packed lower factors, one per attempt group (shared)
    double* Lglob;   // global fallback slice for factors beyond the shared region
    double* Lw;      // the successful attempt's factor
    double* RD;
    double* s1;
    double* s2;
    double* s3;
    double* bb;
    double* xs;
    double* misc;
    int* fidx;
    unsigned* msk;
    const unsigned* cur_mw;  // ballot words of the current free set (build_free_set)
    bool memo_credit;        // credit memoised ccf flops (fast_forward != 2)
    const double* prm;  // global
    const tb_tron_config* cfg;
    int n;
    int t;       // thread index == owned variable
    int tog;     // staging toggle (0 or D); also selects ballot / reduction slots
    int wtog;    // staging toggle of the warp-level PCG (0 or 32)
    BSet act;    // all n variables
    BSet fset;   // current free set, original ownership (rank of variable t)
    BSet cset;   // current free set, compacted ownership (thread p owns rank p)
    int nf;
    long long fl;
    double extrap;
#ifdef TB_PHASES
    long long ph[16];
#endif

    __device__ __forceinline__ void count(long long v) {
        if (COUNT) fl += v;
    }
    __device__ __forceinline__ void sync() { __syncthreads(); }
    __device__ __forceinline__ bool any(bool p) { return __syncthreads_or(p) != 0; }
    __device__ __forceinline__ int cs(int q) const { return q * nf - (q * (q - 1)) / 2; }  // packed column start
    __device__ __forceinline__ double& Lat(int i, int q) { return Lw[cs(q) + (i - q)]; }

    // ------------------------------------------------ ordered reductions
    __device__ __forceinline__ static double dense_sum(const double* b, int cnt) {
        double s = 0.0;
        int j = 0;
#pragma unroll 1
        for (; j + 4 <= cnt; j += 4) {
            const double2 u = *reinterpret_cast<const double2*>(b + j);
            const double2 v = *reinterpret_cast<const double2*>(b + j + 2);
            s += u.x;
            s += u.y;
            s += v.x;
            s += v.y;
        }
#pragma unroll 1
        for (; j < cnt; ++j) s += b[j];
        return s;
    }
    __device__ __forceinline__ double seq_sum(double v, BSet m) {
        double* b = s1 + tog;
        tog ^= D;
        if (m.pos >= 0) b[m.pos] = v;
        sync();
        return dense_sum(b, m.cnt);
    }
    __device__ __forceinline__ void seq_sum2(double a, double c, BSet m, double& sa, double& sc) {
        double* b = s1 + tog;
        double* b2 = s2 + tog;
        tog ^= D;
        if (m.pos >= 0) {
            b[m.pos] = a;
            b2[m.pos] = c;
        }
        sync();
        sa = dense_sum(b, m.cnt);
        sc = dense_sum(b2, m.cnt);
    }
    __device__ __forceinline__ void seq_sum3(double a, double c, double e, BSet m, double& sa, double& sc,
                                             double& se) {
        double* b = s1 + tog;
        double* b2 = s2 + tog;
        double* b3 = s3 + tog;
        tog ^= D;
        if (m.pos >= 0) {
            b[m.pos] = a;
            b2[m.pos] = c;
            b3[m.pos] = e;
        }
        sync();
        sa = dense_sum(b, m.cnt);
        sc = dense_sum(b2, m.cnt);
        se = dense_sum(b3, m.cnt);
    }
    __device__ __forceinline__ double dot(double x, double y, BSet m) {
        count(2 * m.cnt);
        return seq_sum(x * y, m);
    }
    __device__ __forceinline__ double nrm2(double x, BSet m) {
        count(1);
        return sqrt(dot(x, x, m));
    }
    // max / min over the block of non-negative doubles (order-free)
    __device__ __forceinline__ double bmax_nonneg(double v) {
        double* r = misc + BM_RED + (tog ? NW : 0);
        tog ^= D;
        v = warp_max_nonneg(v);
        if ((t & 31) == 0) r[t >> 5] = v;
        sync();
        double m = r[0];
#pragma unroll
        for (int w = 1; w < NW; ++w) m = tb_smax(m, r[w]);
        return m;
    }
    __device__ __forceinline__ double bmin_nonneg(double v) {
        double* r = misc + BM_RED + 2 * NW + (tog ? NW : 0);
        tog ^= D;
        v = warp_min_nonneg(v);
        if ((t & 31) == 0) r[t >> 5] = v;
        sync();
        double m = r[0];
#pragma unroll
        for (int w = 1; w < NW; ++w) m = tb_smin(m, r[w]);
        return m;
    }

    // y = A[m,m] x in original ownership (dense.hpp:104-112, alpha 1, beta 0):
    // column sweep j ascending, zero-skip on x_j, non-members staged as 0
    __device__ __forceinline__ double gemv(double x, BSet m) {
        double* b = s1 + tog;
        tog ^= D;
        if (t < n) b[t] = m.pos >= 0 ? x : 0.0;
        sync();
        double y = 0.0 * 0.0;
        int used = 0;
        if (t < n) {
            const double* Ar = A + t;
#pragma unroll 4
            for (int j = 0; j < n; ++j) {
                const double xj = 1.0 * b[j];
                if (xj != 0.0) {
                    y += xj * Ar[j * D];
                    ++used;
                }
            }
        }
        if (COUNT) {
            int u = 0;
            for (int j = 0; j < n; ++j) u += (1.0 * b[j]) != 0.0;
            fl += 2LL * m.cnt * u;
        }
        (void)used;
        return y;
    }
    // q = B z in compacted ownership, B = A[F,F]
    __device__ __forceinline__ double gemv_c(double z) {
        double* b = s1 + tog;
        tog ^= D;
        if (t < nf) b[t] = z;
        sync();
        double y = 0.0 * 0.0;
        if (t < nf) {
            const double* Ar = A + fidx[t];
#pragma unroll 4
            for (int q = 0; q < nf; ++q) {
                const double zq = 1.0 * b[q];
                if (zq != 0.0) y += zq * Ar[fidx[q] * D];
            }
        }
        if (COUNT) {
            int u = 0;
            for (int q = 0; q < nf; ++q) u += (1.0 * b[q]) != 0.0;
            fl += 2LL * nf * u;
        }
        return y;
    }
    // original ownership (members of the free set) <-> compacted ownership
    __device__ __forceinline__ double to_c(double v) {
        double* b = s1 + tog;
        tog ^= D;
        if (fset.pos >= 0) b[fset.pos] = v;
        sync();
        return t < nf ? b[t] : 0.0;
    }
    __device__ __forceinline__ double to_o(double v) {
        double* b = s1 + tog;
        tog ^= D;
        if (t < nf) b[t] = v;
        sync();
        return fset.pos >= 0 ? b[fset.pos] : 0.0;
    }

    // ------------------------------------------------ tron.hpp primitives
    __device__ __forceinline__ double clip(double x, double l, double u) { return tb_smin(tb_smax(x, l), u); }
    __device__ __forceinline__ double gpstep(double x, double alpha, double w, double l, double u, BSet m) {
        count(2 * m.cnt);
        const double trial = x + alpha * w;
        if (trial < l) return l - x;
        if (trial > u) return u - x;
        return alpha * w;
    }
    __device__ __forceinline__ void breakpt(double x, double w, double l, double u, BSet m, double& bmin,
                                            double& bmax) {
        count(2 * m.cnt);
        double b = 0.0;
        bool has = false;
        if (m.pos >= 0) {
            if (x < u && w > 0.0) { b = (u - x) / w; has = true; }
            else if (x > l && w < 0.0) { b = (l - x) / w; has = true; }
            if (has && !isfinite(b)) has = false;
        }
        if (!any(has)) {
            bmin = 0.0;
            bmax = 0.0;
            return;
        }
        bmin = bmin_nonneg(has ? b : CUDART_INF);
        bmax = bmax_nonneg(has ? b : 0.0);
    }
    __device__ __forceinline__ double pgnorm(double x, double g, double l, double u) {
        double pg = g;
        if (x <= l) pg = tb_smin(g, 0.0);
        else if (x >= u) pg = tb_smax(g, 0.0);
        double v = fabs(pg);
        if (!(t < n) || isnan(v)) v = 0.0;
        return bmax_nonneg(v);
    }
    __device__ __forceinline__ int trqsol(double x, double w, double delta, BSet m, double& sigma) {
        double ptx, ptp, xtx;
        seq_sum3(w * x, w * w, x * x, m, ptx, ptp, xtx);
        count(6 * m.cnt + 8);
        if (ptp == 0.0) return TB_STATUS_ZERO_DIRECTION;
        const double dsq = delta * delta;
        const double rad = sqrt(tb_smax(ptx * ptx + ptp * tb_smax(dsq - xtx, 0.0), 0.0));
        if (ptx > 0.0) sigma = (dsq - xtx) / (ptx + rad);
        else sigma = (rad - ptx) / ptp;
        return 0;
    }
    __device__ __forceinline__ double quad_model(double g, double s, BSet m, double& gs) {
        const double as = gemv(s, m);
        double sas;
        seq_sum2(g * s, s * as, m, gs, sas);
        count(4 * m.cnt + 2);
        return gs + 0.5 * sas;
    }

    // ------------------------------------------------ free set
    // ranks the free variables (ascending index), fills fidx / fset / cset
    __device__ __forceinline__ void build_free_set(bool fr) {
        unsigned* mw = msk + (tog ? NW : 0);
        cur_mw = mw;
        tog ^= D;
        const unsigned b = __ballot_sync(FULL, fr);
        if ((t & 31) == 0) mw[t >> 5] = b;
        sync();
        int before = 0, total = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const int c = __popc(mw[w]);
            if (w < (t >> 5)) before += c;
            total += c;
        }
        const int pos = fr ? before + __popc(b & ((1u << (t & 31)) - 1u)) : -1;
        if (fr) fidx[pos] = t;
        nf = total;
        fset = BSet{total, pos};
        cset = BSet{total, t < total ? t : -1};
        sync();
    }

    // ------------------------------------------------ dense.hpp factorization
    // Shift escalation in parallel (dense.hpp:182-201), like the warp
    // kernel: the reference tries A + a_k I for a_0 = 0, a_{k+1} =
    // max(2 a_k, alpha0) until one factorization succeeds.  Attempts are
    // independent, so the block splits into G groups of GT threads (GT = 32,
    // 64 or 128 >= nf), each running attempt k0 + g on its own packed factor;
    // the first success in k order is the reference's result.  Groups
    // synchronise with __syncwarp (GT <= 32; two 16-lane groups of a warp step
    // through the columns in lockstep) or a named barrier.
    __device__ __forceinline__ void gsync(int gid, int gt) {
        if (gt <= 32) __syncwarp();  // gt = 16: both groups of the warp step in lockstep
        else if (gt == D) __syncthreads();
        else asm volatile("bar.sync %0, %1;" ::"r"(1 + gid), "r"(gt) : "memory");
    }

    // cholesky_left_looking (dense.hpp:138-156) on B = A[F,F] + sh I by one
    // group: thread p computes L(p, j) of column j; the division by d of
    // column j is applied at the start of column j + 1 (one barrier per column).
    // The quotients are branch-free (`quot`, tron_device.cuh); `bad` reports
    // one that left the Markstein range and ccf reruns the round with IEEE
    // divisions (IEEE = true).
    template <bool IEEE>
    __device__ __forceinline__ bool chol_attempt(double sh, double* Lg, const double* Bs, double* slot, int p,
                                                 int gid, int gt, bool valid, long long& fla, bool& bad) {
        const bool rowv = p < nf;
        const double* Ar = A + (rowv ? fidx[p] : 0);
        double* piv = slot;      // [2]
        double* nxt = slot + 2;  // [2]
        double own_prev = 0.0, dprev = 1.0, rprev = 1.0;  // rprev = RN(1 / dprev)
        int csj = 0;                                         // cs(j)
        // gt = 16: a failed (or never valid) group idles until both groups of
        // its warp are done; larger groups leave as soon as their pivot fails
        bool alive = valid;
#pragma unroll 1
        for (int j = 0; j < nf; ++j) {
            const bool row = rowv && p >= j;
            const int pr = row ? p : j;  // row read by this thread (any valid row if idle)
            double lij = row ? (Bs ? Bs[csj + p - j] : Ar[fidx[j] * D]) : 0.0;
            if (p == j) lij += sh;
            int cnt = 0;
            // terms k = 0 .. j-2 (already normalised), ascending; loads first
            const double* Lj = Lg + j;  // L(j, k) = Lj[c_k], c_k = cs(k) - k
            int c = 0, k = 0;
#pragma unroll 1
            for (; k + 4 <= j - 1; k += 4) {
                const int c1 = c + nf - k - 1, c2 = c1 + nf - k - 2, c3 = c2 + nf - k - 3;
                const double l0 = Lj[c], l1 = Lj[c1], l2 = Lj[c2], l3 = Lj[c3];
                const double q0 = Lg[c + pr], q1 = Lg[c1 + pr], q2 = Lg[c2 + pr], q3 = Lg[c3 + pr];
                if (l0 != 0.0) { if (row) lij -= l0 * q0; ++cnt; }
                if (l1 != 0.0) { if (row) lij -= l1 * q1; ++cnt; }
                if (l2 != 0.0) { if (row) lij -= l2 * q2; ++cnt; }
                if (l3 != 0.0) { if (row) lij -= l3 * q3; ++cnt; }
                c = c3 + nf - k - 4;
            }
#pragma unroll 1
            for (; k < j - 1; ++k) {
                const double l0 = Lj[c], q0 = Lg[c + pr];
                if (l0 != 0.0) { if (row) lij -= l0 * q0; ++cnt; }
                c += nf - k - 1;
            }
            // term k = j-1: L(j, j-1) and L(p, j-1) are the quotients of the
            // raw values by d_{j-1} (IEEE, via the correctly rounded reciprocal)
            if (j > 0) {
                const double ljprev = quot<IEEE>(nxt[(j - 1) & 1], dprev, rprev, bad);
                if (row) {
                    own_prev = quot<IEEE>(own_prev, dprev, rprev, bad);
                    Lg[c + p] = own_prev;  // c == cs(j-1) - (j-1)
                }
                if (ljprev != 0.0) {
                    if (row) lij -= ljprev * own_prev;
                    ++cnt;
                }
            }
            if (p == j) piv[j & 1] = lij;
            if (p == j + 1) nxt[j & 1] = lij;
            gsync(gid, gt);
            const double pivot = piv[j & 1];
            const bool ok = pivot > 0.0;
            if (COUNT && alive) fla += 1 + 2LL * (nf - j) * cnt + (ok ? nf - j : 0);
            alive = alive && ok;
            if (gt >= 32) {
                if (!ok) return false;  // the group is a whole warp or more: uniform exit
            } else if (!__any_sync(0xffffffffu, alive)) {
                return false;
            }
            const double d = sqrt(alive ? pivot : 1.0);
            if (p == j) Lg[csj] = d;
            own_prev = lij;
            dprev = d;
            rprev = __drcp_rn(d);  // RN(1/d), the same bits as 1.0 / d
            csj += nf - j;
        }
        return alive;
    }

    // dense.hpp:182-201 shifted_factorize on B.  On success Lw is the factor
    // and RD its reciprocal diagonal.  Returns 0 or FACTORIZATION_FAILED.
#ifndef TB_CCF_MEMO
#define TB_CCF_MEMO 1
#endif
    // Factor memo (as in the warp kernel): ccf is a pure function of A[F,F];
    // while the Hessian is unchanged (the solve loop clears the flag on hess)
    // and the free set repeats, the factor Lw / RD of the previous call is the
    // reference's result again (same shift attempts, same flops).  The factor
    // region is written by ccf alone.  Memo state lives in the block's MISC
    // slots (written by thread 0 before a barrier, read by every thread).
    __device__ __forceinline__ bool memo_hit() {
        const int* flag = reinterpret_cast<const int*>(misc + BM_MEMO);
        const unsigned* words = reinterpret_cast<const unsigned*>(misc + BM_MEMO + 2);
        bool hit = *flag != 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) hit = hit && words[w] == cur_mw[w];
        return hit;
    }
    __device__ __forceinline__ void memo_store(long long flops) {  // before the barrier that ends ccf
        if (t == 0) {
            *reinterpret_cast<int*>(misc + BM_MEMO) = 1;
            *reinterpret_cast<long long*>(misc + BM_MEMO + 1) = flops;
            unsigned* words = reinterpret_cast<unsigned*>(misc + BM_MEMO + 2);
#pragma unroll
            for (int w = 0; w < NW; ++w) words[w] = cur_mw[w];
        }
    }
    __device__ __forceinline__ void memo_clear() {  // thread 0; ordered by later barriers
        if (t == 0) *reinterpret_cast<int*>(misc + BM_MEMO) = 0;
    }

    __device__ __forceinline__ int ccf(double& shift) {
        if (TB_CCF_MEMO && memo_hit()) {
            if (memo_credit) count(*reinterpret_cast<const long long*>(misc + BM_MEMO + 1));
            return 0;
        }
        const long long fl0 = fl;
        // 16-lane groups (4 attempts at once) pay at D = 64 (d = 24: -10 %, d = 64: -3 %);
        // at D = 128 eight lockstep groups cost more than they save (+2 %)
        const int gt = (D == 32 && nf <= 8)    ? 8
                       : (nf <= 16 && D <= 64) ? 16
                       : (nf <= 32 ? 32 : (nf <= 64 && D > 64 ? 64 : D));
        const int G = D / gt;
        const int gid = t / gt, p = t % gt;
        const int lpg = ((nf * (nf + 1)) / 2 + 1) & ~1;
        // factors in the shared region when they fit, else the global slice
        double* Lbase = G * lpg <= SL::LP ? L : Lglob;
        double* Lg = Lbase + gid * lpg;
        // B = A[F,F] (lower triangle) staged once per call behind the G
        // factors when it fits: every attempt then reads shared memory
        double* Bs = (Lbase == L && (G + 1) * lpg <= SL::LP) ? L + G * lpg : nullptr;
        double dg = 0.0, ma = 0.0;
        if (t < nf) {
            const double* Ar = A + fidx[t];
            dg = fabs(Ar[fidx[t] * D]);
            if (isnan(dg)) dg = 0.0;
#pragma unroll 4
            for (int q = 0; q < nf; ++q) {
                const double a = Ar[fidx[q] * D];
                if (Bs && q <= t) Bs[cs(q) + t - q] = a;
                const double v = fabs(a);
                if (!isnan(v)) ma = fmax(ma, v);
            }
        }
        const double max_diag = bmax_nonneg(dg);
        const double max_abs = bmax_nonneg(ma);
        const double alpha0 = tb_smax(1e-3 * max_diag, 1e-8);
        const double cap = 1e8 * tb_smax(1.0, max_abs);
        int* gok = reinterpret_cast<int*>(misc + BM_GOK);
        long long* gfl = reinterpret_cast<long long*>(misc + BM_GFL);
        double base = 0.0;  // a_{k0}
#pragma unroll 1
        for (int k0 = 0;; k0 += G) {
            const double sh = tb_shift_ahead(base, alpha0, gid);  // a_{k0+gid}
            const bool valid = (k0 + gid == 0) || (sh <= cap);
            long long fla = 0;
            bool ok = false, bad = false;
            if (valid || gt < 32) {  // sub-warp groups share a warp: all enter the lockstep loop
                TB_PH_BEGIN(11)
                ok = chol_attempt<false>(sh, Lg, Bs, misc + BM_GRP + 4 * gid, p, gid, gt, valid, fla, bad);
                TB_PH_END(*this, 11)
            }
            if (__syncthreads_or(bad)) {  // rare: rerun the round with IEEE divisions
                fla = 0;
                ok = false;
                if (valid || gt < 32)
                    ok = chol_attempt<true>(sh, Lg, Bs, misc + BM_GRP + 4 * gid, p, gid, gt, valid, fla, bad);
            }
            if (p == 0) {
                gok[gid] = ok ? 1 : (valid ? 0 : -1);
                if (COUNT) gfl[gid] = fla;
            }
            sync();
            int winner = -1;
            bool all_valid = true;
            for (int q = 0; q < G; ++q) {
                const int v = gok[q];
                if (v == 1 && winner < 0) winner = q;
                if (v < 0) all_valid = false;
            }
            if (COUNT) {
                const int last = winner >= 0 ? winner : G - 1;
                for (int q = 0; q <= last; ++q)
                    if (gok[q] >= 0) count(gfl[q] + ((q < winner || winner < 0) ? 1 : 0));
            }
            if (winner >= 0) {
                shift = tb_shift_ahead(base, alpha0, winner);
                Lw = Lbase + winner * lpg;
                if (t < nf) RD[t] = __drcp_rn(Lat(t, t));
                if (TB_CCF_MEMO) memo_store(fl - fl0);
                sync();
                return 0;
            }
            // no success among attempts k0..k0+G-1: the reference throws at
            // the first a_k > cap (all earlier attempts failed)
            if (!all_valid) return TB_STATUS_FACTORIZATION_FAILED;
            base = tb_shift_ahead(base, alpha0, G);
            sync();  // gok / group slots are rewritten by the next round
        }
    }

    // forward solve L b = rhs in compacted ownership (column sweep).  The
    // quotients take the branch-free Markstein form (tron_device.cuh `quot`);
    // one barrier-vote at the end sends a solve that met an out-of-range
    // quotient through the IEEE divisions again (same results as div_rcp).
    template <bool IEEE>
    __device__ __forceinline__ double trsv_fwd_core(double b, bool& bad) {
        const int p = t;
        double s = p < nf ? b : 0.0;
#pragma unroll 1
        for (int j = 0; j < nf; ++j) {
            if (p == j) {
                s = quot<IEEE>(s, Lat(j, j), RD[j], bad);
                bb[j] = s;
            }
            sync();
            const double q = bb[j];
            if (p > j && p < nf) s -= Lat(p, j) * q;
        }
        return s;
    }
    __device__ __forceinline__ double trsv_fwd(double b) {
        bool bad = false;
        const double s = trsv_fwd_core<false>(b, bad);
        if (!__syncthreads_or(bad)) return s;
        return trsv_fwd_core<true>(b, bad);
    }
    // backward solve L^T b = rhs (dense.hpp:229-235): for i descending,
    // s = b_i - sum_{j > i ascending} L(j,i) b_j, serial on warp 0 (all lanes
    // compute the same values)
    __device__ __forceinline__ double trsv_bwd(double b) {
        double* in = s1 + tog;
        tog ^= D;
        if (t < nf) in[t] = b;
        sync();
        if (t < 32) bwd_solve(in);
        sync();
        return t < nf ? bb[t] : 0.0;
    }
    // the serial backward recurrence, run by warp 0 (lanes compute the same
    // values, so `bad` is warp-uniform); results in bb[0..nf-1]
    __device__ __forceinline__ void bwd_solve(const double* in) {
        bool bad = false;
        bwd_core<false>(in, bad);
        if (bad) bwd_core<true>(in, bad);
    }
    template <bool IEEE>
    __device__ __forceinline__ void bwd_core(const double* in, bool& bad) {
        double last = 0.0;
#pragma unroll 1
        for (int i = nf - 1; i >= 0; --i) {
            const double* Lc = Lw + cs(i) - i;  // L(j, i) = Lc[j]
            double s = in[i];
            if (i + 1 < nf) s -= Lc[i + 1] * last;
            int j = i + 2;
#pragma unroll 1
            for (; j + 4 <= nf; j += 4) {
                const double p0 = Lc[j] * bb[j];
                const double p1 = Lc[j + 1] * bb[j + 1];
                const double p2 = Lc[j + 2] * bb[j + 2];
                const double p3 = Lc[j + 3] * bb[j + 3];
                s -= p0;
                s -= p1;
                s -= p2;
                s -= p3;
            }
#pragma unroll 1
            for (; j < nf; ++j) s -= Lc[j] * bb[j];
            last = quot<IEEE>(s, Lc[i], RD[i], bad);
            if (t == 0) bb[i] = last;
            __syncwarp();
        }
    }

    // ---------------------------------- warp-level PCG pieces (nf <= 32)
    // Run by warp 0 only (lane p owns free rank p); shuffles and __syncwarp,
    // no block barrier.  Same operations in the same order as the block forms.
    // Staging (s1, s2, s3 are idle while the other warps wait): s1[0,64) sums,
    // s2[0,64) / s3[0,64) the 2nd / 3rd sums, s2[64,128) backward-solve input,
    // s3[64,128) gemv input; each toggled by wtog.
    __device__ __forceinline__ double wsum(double v) {
        double* b = s1 + wtog;
        wtog ^= 32;
        if (t < nf) b[t] = v;
        __syncwarp();
        return dense_sum(b, nf);
    }
    __device__ __forceinline__ void wsum3(double a, double c, double e, double& sa, double& sc, double& se) {
        double* b = s1 + wtog;
        double* b2 = s2 + wtog;
        double* b3 = s3 + wtog;
        wtog ^= 32;
        if (t < nf) {
            b[t] = a;
            b2[t] = c;
            b3[t] = e;
        }
        __syncwarp();
        sa = dense_sum(b, nf);
        sc = dense_sum(b2, nf);
        se = dense_sum(b3, nf);
    }
    __device__ __forceinline__ double wdot(double x, double y) {
        count(2 * nf);
        return wsum(x * y);
    }
    template <bool IEEE>
    __device__ __forceinline__ double wtrsv_fwd_core(double b, bool& bad) {
        const int p = t;
        double s = p < nf ? b : 0.0;
#pragma unroll 1
        for (int j = 0; j < nf; ++j) {
            const double q = quot<IEEE>(__shfl_sync(FULL, s, j), Lat(j, j), RD[j], bad);
            if (p == j) s = q;
            else if (p > j && p < nf) s -= Lat(p, j) * q;
        }
        return s;
    }
    __device__ __forceinline__ double wtrsv_fwd(double b) {  // warp 0; `bad` is warp-uniform
        bool bad = false;
        const double s = wtrsv_fwd_core<false>(b, bad);
        return bad ? wtrsv_fwd_core<true>(b, bad) : s;
    }
    __device__ __forceinline__ double wtrsv_bwd(double b) {
        double* in = s2 + 64 + wtog;
        wtog ^= 32;
        if (t < nf) in[t] = b;
        __syncwarp();
        bwd_solve(in);
        return t < nf ? bb[t] : 0.0;
    }
    __device__ __forceinline__ double wgemv_c(double z) {
        double* b = s3 + 64 + wtog;
        wtog ^= 32;
        if (t < nf) b[t] = z;
        __syncwarp();
        double y = 0.0 * 0.0;
        int u = 0;
        if (t < nf) {
            const double* Ar = A + fidx[t];
#pragma unroll 4
            for (int q = 0; q < nf; ++q) {
                const double zq = 1.0 * b[q];
                if (zq != 0.0) y += zq * Ar[fidx[q] * D];
            }
        }
        if (COUNT) {
            for (int q = 0; q < nf; ++q) u += (1.0 * b[q]) != 0.0;
            fl += 2LL * nf * u;
        }
        return y;
    }
    __device__ __forceinline__ int wtrqsol(double x, double w, double delta, double& sigma) {
        double ptx, ptp, xtx;
        wsum3(w * x, w * w, x * x, ptx, ptp, xtx);
        count(6 * nf + 8);
        if (ptp == 0.0) return TB_STATUS_ZERO_DIRECTION;
        const double dsq = delta * delta;
        const double rad = sqrt(tb_smax(ptx * ptx + ptp * tb_smax(dsq - xtx, 0.0), 0.0));
        if (ptx > 0.0) sigma = (dsq - xtx) / (ptx + rad);
        else sigma = (rad - ptx) / ptp;
        return 0;
    }
    // tron.hpp:290-344 on warp 0
    __device__ __forceinline__ int precond_cg_w(double gfree, double delta, double& step, int& cg_status,
                                                int& iters) {
        const long long nf2 = (long long)nf * nf;
        double w = 0.0;
        count(nf);
        const double bhat = wtrsv_fwd(gfree * -1.0);
        count(nf2);
        count(1);
        const double bnorm = sqrt(wdot(bhat, bhat));
        iters = 0;
        if (bnorm == 0.0) {
            step = 0.0;
            cg_status = 0;
            return 0;
        }
        double r = bhat, p = r;
        double rho = wdot(r, r);
        cg_status = 3;
#pragma unroll 1
        for (int k = 1; k <= nf; ++k) {
            iters = k;
            const double z = wtrsv_bwd(p);
            double q = wgemv_c(z);
            q = wtrsv_fwd(q);
            count(2 * nf2);
            const double ptq = wdot(p, q);
            double sigma;
            const int rc = wtrqsol(w, p, delta, sigma);
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
            const double rtr = wdot(r, r);
            count(2);
            if (sqrt(rtr) <= cfg->cg_tol * bnorm) {
                cg_status = 0;
                break;
            }
            const double beta = rtr / rho;
            p = beta * p;
            p += 1.0 * r;
            count(3 * nf + 1);
            rho = rtr;
        }
        step = wtrsv_bwd(w);
        count(nf2);
        return 0;
    }

    // ------------------------------------------------ tron.hpp:290-344
    // Steihaug PCG in compacted ownership (thread p < nf owns free rank p)
    __device__ __forceinline__ int precond_cg(double gfree, double delta, double& step, int& cg_status, int& iters) {
        const long long nf2 = (long long)nf * nf;
        const BSet C = cset;
        double w = 0.0;
        count(nf);
        const double bhat = trsv_fwd(gfree * -1.0);
        count(nf2);
        const double bnorm = nrm2(bhat, C);
        iters = 0;
        if (bnorm == 0.0) {
            step = 0.0;
            cg_status = 0;
            return 0;
        }
        double r = bhat, p = r;
        double rho = dot(r, r, C);
        cg_status = 3;
#pragma unroll 1
        for (int k = 1; k <= nf; ++k) {
            iters = k;
            TB_PH_BEGIN(9)
            const double z = trsv_bwd(p);
            TB_PH_END(*this, 9)
            TB_PH_BEGIN(10)
            double q = gemv_c(z);
            TB_PH_END(*this, 10)
            TB_PH_BEGIN(8)
            q = trsv_fwd(q);
            TB_PH_END(*this, 8)
            count(2 * nf2);
            const double ptq = dot(p, q, C);
            double sigma;
            const int rc = trqsol(w, p, delta, C, sigma);
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
            const double rtr = dot(r, r, C);
            count(2);
            if (sqrt(rtr) <= cfg->cg_tol * bnorm) {
                cg_status = 0;
                break;
            }
            const double beta = rtr / rho;
            p = beta * p;
            p += 1.0 * r;
            count(3 * nf + 1);
            rho = rtr;
        }
        step = trsv_bwd(w);
        count(nf2);
        return 0;
    }

    // tron.hpp:354-374 on the free set (original ownership)
    __device__ __forceinline__ double line_search(double x, double l, double u, double g, double w) {
        const BSet F = fset;
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
            count(2 * F.cnt + 1);
            if (q <= cfg->mu0 * gs) search = false;
            else beta *= cfg->interp_factor;
        }
        if (beta < 1.0 && beta < bmin) beta = bmin;
        count(2 * F.cnt);
        return clip(x + beta * w, l, u);
    }

    // tron.hpp:201-250 (same state machine as the warp kernel)
    __device__ __forceinline__ int cauchy(double x, double g, double l, double u, double delta, double alpha_start,
                                          double& alpha_out, double& s) {
        const BSet m = act;
        const double radius = cfg->mu1 * delta;
        double alpha = alpha_start;
        const double mg = -1.0 * g;
        count(n);
        double bmin, bmax;
        breakpt(x, mg, l, u, m, bmin, bmax);
        int mode = 0;
        double alpha_good = alpha;
#pragma unroll 1
        for (;;) {
            s = gpstep(x, -alpha, g, l, u, m);
            const double nr = nrm2(s, m);
            const bool evalq = mode == 0 ? !(nr > radius) : (nr <= radius);
            bool qge = false;
            if (evalq) {
                double gs;
                const double q = quad_model(g, s, m, gs);
                if (!isfinite(q)) return TB_STATUS_EVALUATION_ERROR;
                count(2 * n + 1);
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
                const bool srch = evalq ? qge : true;
                if (!srch || !(alpha > 1e-30)) break;
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
            s = gpstep(x, -alpha, g, l, u, m);
        }
        alpha_out = alpha;
        return 0;
    }

    // tron.hpp:394-447
    __device__ __forceinline__ int subspace_step(double x0, double g, double l, double u, double delta, double cs_,
                                                 double& xout, double& sout, long long& cg_total) {
        xout = clip(x0 + 1.0 * cs_, l, u);
        count(2 * n);
        double s = xout - x0;
        count(n);
        double w = gemv(s, act);
        cg_total = 0;
#pragma unroll 1
        for (int faces = 0; faces < n; ++faces) {
            const bool fr = t < n && l < xout && xout < u;
            build_free_set(fr);
            if (nf == 0) break;
            double shift;
            TB_PH_BEGIN(2)
            int rc = ccf(shift);
            TB_PH_END(*this, 2)
            if (rc) return rc;
            if (any(t < nf && Lat(t, t) == 0.0)) return TB_STATUS_SINGULAR_FACTOR;
            const double gfree = w + g;
            count(nf);
            const double gfnorm = nrm2(g, fset);
            double step_c;
            int cgs, its;
            TB_PH_BEGIN(3)
            const double gc = to_c(gfree);
            if (nf <= 32) {  // warp 0 alone, no block barriers
                int* res = reinterpret_cast<int*>(misc + BM_PCG);
                if (t < 32) {
                    rc = precond_cg_w(gc, delta, step_c, cgs, its);
                    if (t == 0) {
                        res[0] = rc;
                        res[1] = cgs;
                        res[2] = its;
                    }
                }
                sync();
                rc = res[0];
                cgs = res[1];
                its = res[2];
            } else {
                rc = precond_cg(gc, delta, step_c, cgs, its);
            }
            TB_PH_END(*this, 3)
            if (rc) return rc;
            cg_total += its;
            const double step = to_o(step_c);
            TB_PH_BEGIN(4)
            const double xn = line_search(xout, l, u, gfree, step);
            TB_PH_END(*this, 4)
            if (fr) {
                s += xn - xout;
                xout = xn;
            }
            count(2 * nf);
            w = gemv(s, act);
            const double tt = w + g;
            const double gfnormf = seq_sum(tt * tt, fset);
            count(3 * nf + 2);
            if (sqrt(gfnormf) <= cfg->cg_tol * gfnorm) break;
            if (cgs == 1 || cgs == 3) break;
        }
        sout = s;
        return 0;
    }
};

// ------------------------------------------------------------ families
// Same tb_families.h expressions as the warp kernel's DevFamily; parameters
// are read from global memory.  The branch family (d = 4 / 6) never gets here.
template <int FAM, int D, bool ASMEM, bool COUNT>
struct BlkFamily {
    using B = Blk<D, ASMEM, COUNT>;
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;

    __device__ __forceinline__ void prepare(B& W, double x) {
        const int t = W.t, n = W.n;
        const bool act = t < n;
        if (act) W.xs[t] = x;
        W.sync();
        const double* prm = W.prm;
        if (FAM == TB_FAMILY_BOXQP) {
            if (act) {
                c0 = x - prm[(long)n * n + t];
                c1 = tb_boxqp_hd_i(W.xs, prm, n, t);
            }
        } else if (FAM == TB_FAMILY_NCVX) {
            if (act) {
                const double* c = prm + (long)n * (n + 1) / 2;
                c0 = x - c[t];
                c1 = tb_ncvx_he_i(W.xs, prm, n, t);
                tb_sincos(x, &c2, &c3);
            }
        }
    }
    __device__ __forceinline__ double f(B& W) {
        const int t = W.t, n = W.n;
        const double* prm = W.prm;
        if (FAM == TB_FAMILY_HS45) return tb_hs45_f(W.xs, n);
        if (FAM == TB_FAMILY_BOXQP) return 0.5 * W.seq_sum(c0 * c1, W.act);
        const double* k = prm + (long)n * (n + 1) / 2 + n;
        const double* a = k + n;
        const double e2 = c0 * c0;
        double q, quart, sn;
        const double kq = t < n ? k[t] * (e2 * e2) : 0.0;
        const double as = t < n ? a[t] * c2 : 0.0;
        W.seq_sum3(c0 * c1, kq, as, W.act, q, quart, sn);
        return (0.5 * q + 0.25 * quart) + sn;
    }
    __device__ __forceinline__ double grad(B& W) {
        const int t = W.t, n = W.n;
        if (t >= n) return 0.0;
        const double* prm = W.prm;
        if (FAM == TB_FAMILY_HS45) return tb_hs45_grad_i(W.xs, n, t);
        if (FAM == TB_FAMILY_BOXQP) return c1;
        const double* k = prm + (long)n * (n + 1) / 2 + n;
        const double* a = k + n;
        const double e3 = (c0 * c0) * c0;
        return (c1 + k[t] * e3) + a[t] * c3;
    }
    // row t of the Hessian into A[t + j*D].  The off-diagonal entries of
    // NCVX (the packed H) and the whole BOXQP Hessian do not depend on x:
    // after the first evaluation of a problem only the NCVX diagonal is
    // rewritten (same expressions, same bits; the block's A slice is written
    // by hess alone, and the family object lives for one problem).
    bool const_part = false;
    __device__ __forceinline__ void hess(B& W) {
        const int t = W.t, n = W.n;
        const double* prm = W.prm;
        double* Ar = W.A + t;
        if (t < n) {
            if (FAM == TB_FAMILY_HS45) {
                for (int j = 0; j < n; ++j) Ar[j * D] = tb_hs45_hess(W.xs, n, t, j);
            } else if (FAM == TB_FAMILY_BOXQP) {
                if (!const_part)
                    for (int j = 0; j < n; ++j) Ar[j * D] = tb_boxqp_hess(prm, n, t, j);
            } else {
                const double* k = prm + (long)n * (n + 1) / 2 + n;
                const double* a = k + n;
                if (!const_part)
                    for (int j = 0; j < n; ++j)
                        if (j != t) Ar[j * D] = tb_ncvx_H(prm, n, t, j);
                Ar[t * D] = (tb_ncvx_H(prm, n, t, t) + (3.0 * k[t]) * (c0 * c0)) - a[t] * c2;
            }
        }
        const_part = TB_HESS_CONST_PART;
        W.sync();
    }
};

// tron.hpp:453-549 solve(), one problem per block, persistent over the batch.
// a.ws: the work counter (first 256 bytes), then one D x D Hessian slice per
// block (global variant).
constexpr size_t kBlkWsHeader = 256;
template <int D>
struct BlkMinBlocks {
    static constexpr int value = D >= 128 ? TB_BLK_MIN128 : (D >= 64 ? TB_BLK_MIN64 : TB_BLK_MIN32);
};
// ws = header | A slices (grid x D^2, global-A variant) | factor fallback
// slices (grid x LPFULL, D = 128 only)
template <int D>
__device__ __forceinline__ double* blk_lglob(const KernelArgs& a, bool asmem) {
    double* base = reinterpret_cast<double*>(static_cast<char*>(a.ws) + kBlkWsHeader);
    if (!asmem) base += (size_t)gridDim.x * D * D;
    return base + (size_t)blockIdx.x * (D * (D + 1) / 2);
}

template <int FAM, int D, bool ASMEM, bool COUNT, bool ORD = false>
__global__ void __launch_bounds__(D, BlkMinBlocks<D>::value) tron_block_kernel(const __grid_constant__ KernelArgs a) {
    extern __shared__ double smem[];
    using SL = BlkLayout<D, ASMEM>;
    Blk<D, ASMEM, COUNT> W;
    unsigned* work = static_cast<unsigned*>(a.ws);
    W.A = ASMEM ? smem + SL::AS
                : reinterpret_cast<double*>(static_cast<char*>(a.ws) + kBlkWsHeader) + (size_t)blockIdx.x * D * D;
    W.L = smem + SL::L;
    W.Lw = W.L;
    W.Lglob = SL::LP < SL::LPFULL ? blk_lglob<D>(a, ASMEM) : nullptr;
    W.RD = smem + SL::RD;
    W.s1 = smem + SL::S1;
    W.s2 = smem + SL::S2;
    W.s3 = smem + SL::S3;
    W.bb = smem + SL::BB;
    W.xs = smem + SL::XS;
    W.misc = smem + SL::MISC;
    W.fidx = reinterpret_cast<int*>(smem + SL::FIDX);
    W.msk = reinterpret_cast<unsigned*>(smem + SL::MSK);
    W.cfg = &a.cfg;
    W.extrap = a.extrap;
    W.n = a.n;
    W.t = threadIdx.x;
    W.tog = 0;
    W.wtog = 0;
    W.nf = 0;
    W.memo_credit = a.fast_forward != 2;
    const int n = a.n;
    const int t = W.t;
    const bool act = t < n;
    W.act = BSet{n, act ? t : -1};
    const tb_tron_config& cfg = a.cfg;
    unsigned* pid_slot = reinterpret_cast<unsigned*>(W.misc + BM_PID);

#pragma unroll 1
    for (;;) {
        if (t == 0) *pid_slot = atomicAdd(work, 1u);
        __syncthreads();
        const long long k = *pid_slot;
        __syncthreads();
        if (k >= a.count) break;
        const long long pid = ORD ? (long long)a.order[k] : k;  // ORD: ranked work items (tron_order.cu)
        W.memo_clear();  // a new problem: no memoised factor (ordered by the barriers before ccf)
        const unsigned long long t_start = globaltimer();
        W.fl = 0;
#ifdef TB_PHASES
        for (int k = 0; k < 16; ++k) W.ph[k] = 0;
        const long long tb_ph_total0 = clock64();
#endif
        W.prm = a.prm ? a.prm + pid * a.stride : nullptr;
        BlkFamily<FAM, D, ASMEM, COUNT> fam;
        const double l = act ? a.lo[pid * n + t] : 0.0;
        const double u = act ? a.up[pid * n + t] : 0.0;
        double x = act ? a.x0[pid * n + t] : 0.0;

        // block-uniform loop state in shared memory, one copy per warp (warps
        // run apart between barriers; registers set residency).  The counters
        // (read-modify-write) are updated by lane 0 of each warp and read by
        // thread 0; every lane stores the same value into the other slots, and
        // f / delta_in / alpha_in, read by every lane before they are rewritten
        // in the same pass, are rewritten after a __syncwarp
        const bool wl0 = (t & 31) == 0;
        double* sc = W.misc + BM_SC + 8 * (t >> 5);
        long long& cg_iterations = reinterpret_cast<long long*>(sc)[0];
        long long& f_evals = reinterpret_cast<long long*>(sc)[1];
        double& f = sc[2];
        double& pg = sc[3];
        int& iterations = reinterpret_cast<int*>(sc + 4)[0];
        int& status = reinterpret_cast<int*>(sc + 4)[1];
        double& delta_in = sc[5];
        double& alpha_in = sc[6];
        status = TB_STATUS_ITER_LIMIT;
        iterations = 0;
        cg_iterations = 0;
        f_evals = 0;
        f = 0.0;
        pg = 0.0;

        if (W.any(act && !(l <= u))) {
            status = TB_STATUS_INVALID_BOUNDS;
        } else {
            const double kEta1 = 0.25, kEta2 = 0.75;
            x = W.clip(x, l, u);
            double xe = x;
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
                TB_PH_END(W, 6)
                W.count(tb_family_flops(FAM, n, 0));
                if (wl0) ++f_evals;
                bool take = iter == 0;
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
                    take = actred > cfg.eta0 * prered;
                    if (take) {
                        x = xe;
                        __syncwarp();  // every lane of the warp has read f
                        f = f_trial;
                        need_hessian = true;
                    }
                } else {
                    f = fe;
                }
                if (take) {
                    g = fam.grad(W);
                    W.count(tb_family_flops(FAM, n, 1));
                    pg = W.pgnorm(x, g, l, u);
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
                    if (a.fast_forward && !take && iter >= 2 && delta == delta_in && alpha_c == alpha_in) {
                        const long long rem = cfg.max_iter - iter;
                        if (wl0) {
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
                if (need_hessian) {
                    TB_PH_BEGIN(0)
                    fam.hess(W);
                    TB_PH_END(W, 0)
                    W.count(tb_family_flops(FAM, n, 2));
                    need_hessian = false;
                    W.memo_clear();  // a new Hessian: the memoised factor is stale
                }
                fl_iter0 = W.fl;
                __syncwarp();  // every lane of the warp has read delta_in / alpha_in
                delta_in = delta;
                alpha_in = alpha_c;
                double cs, alpha_new;
                TB_PH_BEGIN(1)
                int rc = W.cauchy(x, g, l, u, delta, alpha_c, alpha_new, cs);
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
                    status = rc;
                    break;
                }
                if (wl0) cg_iterations += cg_its;
            }
        }
#ifdef TB_PHASES
        W.ph[7] = clock64() - tb_ph_total0;
        if (t == 0)
            for (int k = 0; k < 16; ++k) atomicAdd(&g_phase_cycles[k], (unsigned long long)W.ph[k]);
#endif
        __syncwarp();  // every lane's last store of the loop scalars before thread 0 reports them
        if (act && a.x_star) a.x_star[pid * n + t] = x;
        if (t == 0) {
            if (a.f_star) a.f_star[pid] = f;
            if (a.pg_norm) a.pg_norm[pid] = pg;
            if (a.status) a.status[pid] = status;
            if (a.iterations) a.iterations[pid] = iterations;
            if (a.cg_iterations) a.cg_iterations[pid] = cg_iterations;
            if (a.f_evals) a.f_evals[pid] = f_evals;
            if (a.flops) a.flops[pid] = W.fl;
            if (a.wall_time) a.wall_time[pid] = 1e-9 * (double)(globaltimer() - t_start);
        }
        __syncthreads();
    }
}

}  // namespace tbdev
