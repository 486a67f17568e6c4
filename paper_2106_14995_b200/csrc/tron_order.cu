// tron_order.cu — launch order of a batch: longest-expected-first.
//
// A one-shot launch ends with its slowest problem, and a problem that starts
// late in the launch (blocks are dispatched in index order) finishes late.
// For the branch family the number of TRON iterations a problem needs is
// predicted well by the projected-gradient inf-norm at its clipped start
// point -- the quantity solve() tests first (tron.hpp:473-483): on C2 every
// problem that needs >= 100 iterations is in the top quarter of that ranking,
// and the ranked launch runs as fast as one sorted by the oracle's actual
// iteration counts (the host decides where ranking pays).  So
// the library ranks the batch by it on the device and launches problem
// order[k] as the k-th block / thread / work item.  Results are per problem
// and written at the problem's own index: the order changes WHEN a problem
// is solved, never what is computed (every SolveReport field is identical).
//
// Three small kernels: a key per problem (one thread: clip, gradient,
// projected-gradient norm -> a log-scale bucket, block-local histogram), an
// exclusive scan of the bucket counts (descending keys first), and a scatter
// (atomic slot per bucket; the order inside a bucket is arbitrary).
#include <cuda_runtime.h>
#include <stdint.h>

#include "tb_families.h"
#include "tron_launch.h"

namespace tbdev {
namespace {

constexpr int kBuckets = 4096;  // 32 per octave over 2^-64 .. 2^64 (few ties: a stable schedule)
constexpr int kKeyBlock = 128;
constexpr int kScanThreads = 1024;

// bucket 0 = largest key; NaN / inf first
__device__ __forceinline__ unsigned order_bucket(double pg) {
    if (!(pg == pg)) return 0;
    const long long b = (long long)((unsigned long long)__double_as_longlong(pg) >> 47);  // exponent + 5 bits
    const long long lo = (1023LL - 64) << 5, hi = lo + kBuckets - 1;
    const long long v = b < lo ? lo : (b > hi ? hi : b);
    return (unsigned)(hi - v);
}

// projected-gradient inf-norm (tron.hpp:112-121) at clip(x0) of one problem
template <int FAM, int D>
__device__ double start_pg(const KernelArgs& a, long long pid) {
    const int n = a.n;
    double x[D];
    const double* lo = a.lo + pid * n;
    const double* up = a.up + pid * n;
    const double* prm = a.prm ? a.prm + pid * a.stride : nullptr;
    for (int i = 0; i < n; ++i) x[i] = tb_smin(tb_smax(a.x0[pid * n + i], lo[i]), up[i]);
    double pg = 0.0;
    auto add = [&](int i, double g) {
        if (x[i] <= lo[i]) g = tb_smin(g, 0.0);
        else if (x[i] >= up[i]) g = tb_smax(g, 0.0);
        const double v = fabs(g);
        if (v == v) pg = tb_smax(pg, v);
    };
    if (FAM == TB_FAMILY_BRANCH) {
        tb_branch_ctx c;
        tb_branch_ctx_init(x, prm, n, &c);
        for (int i = 0; i < n; ++i) add(i, tb_br_grad(&c, n, i));
    } else {
        for (int i = 0; i < n; ++i) {
            double g;
            if (FAM == TB_FAMILY_HS45) g = tb_hs45_grad_i(x, n, i);
            else if (FAM == TB_FAMILY_BOXQP) g = tb_boxqp_grad_i(x, prm, n, i);
            else g = tb_ncvx_grad_i(x, prm, n, i);
            add(i, g);
        }
    }
    return pg;
}

template <int FAM, int D>
__global__ void __launch_bounds__(kKeyBlock) order_key_kernel(const __grid_constant__ KernelArgs a,
                                                             uint32_t* bucket, uint32_t* hist) {
    __shared__ uint32_t h[kBuckets];
    for (int i = threadIdx.x; i < kBuckets; i += kKeyBlock) h[i] = 0;
    __syncthreads();
    const long long pid = blockIdx.x * (long long)kKeyBlock + threadIdx.x;
    if (pid < a.count) {
        const unsigned b = order_bucket(start_pg<FAM, D>(a, pid));
        bucket[pid] = b;
        atomicAdd(&h[b], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kBuckets; i += kKeyBlock)
        if (h[i]) atomicAdd(&hist[i], h[i]);
}

// exclusive scan of the bucket counts (one block; each thread owns a run of
// kBuckets / kScanThreads consecutive buckets)
__global__ void __launch_bounds__(kScanThreads) order_scan_kernel(const uint32_t* hist, uint32_t* offs) {
    constexpr int R = kBuckets / kScanThreads;
    __shared__ uint32_t s[kScanThreads];
    const int t = threadIdx.x;
    uint32_t v[R], run = 0;
    for (int k = 0; k < R; ++k) {
        v[k] = hist[t * R + k];
        run += v[k];
    }
    s[t] = run;
    __syncthreads();
    for (int d = 1; d < kScanThreads; d <<= 1) {
        const uint32_t add = t >= d ? s[t - d] : 0u;
        __syncthreads();
        s[t] += add;
        __syncthreads();
    }
    uint32_t base = s[t] - run;
    for (int k = 0; k < R; ++k) {
        offs[t * R + k] = base;
        base += v[k];
    }
}

__global__ void order_scatter_kernel(const uint32_t* bucket, uint32_t* offs, uint32_t* order, long long count) {
    const long long pid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (pid < count) order[atomicAdd(&offs[bucket[pid]], 1u)] = (uint32_t)pid;
}

template <int FAM, int D>
cudaError_t launch_key(const KernelArgs& a, uint32_t* bucket, uint32_t* hist, cudaStream_t st) {
    order_key_kernel<FAM, D><<<(unsigned)((a.count + kKeyBlock - 1) / kKeyBlock), kKeyBlock, 0, st>>>(a, bucket, hist);
    return cudaGetLastError();
}

template <int FAM>
cudaError_t launch_key_fam(const KernelArgs& a, uint32_t* bucket, uint32_t* hist, cudaStream_t st) {
    const int n = a.n;
    if (FAM == TB_FAMILY_BRANCH) return n == 4 ? launch_key<FAM, 4>(a, bucket, hist, st) : launch_key<FAM, 6>(a, bucket, hist, st);
    if (n <= 8) return launch_key<FAM, 8>(a, bucket, hist, st);
    if (n <= 32) return launch_key<FAM, 32>(a, bucket, hist, st);
    return launch_key<FAM, 128>(a, bucket, hist, st);
}

}  // namespace

size_t order_ws_bytes(long long count) { return sizeof(uint32_t) * (2 * (size_t)kBuckets + 2 * (size_t)count); }

// order[k] = the problem launched k-th (descending start projected-gradient
// norm); `ws` holds order_ws_bytes(a.count).  Stream-ordered on `st`.
cudaError_t launch_order(int family, const KernelArgs& a, void* ws, cudaStream_t st, const uint32_t** order_out) {
    uint32_t* hist = static_cast<uint32_t*>(ws);
    uint32_t* offs = hist + kBuckets;
    uint32_t* bucket = offs + kBuckets;
    uint32_t* order = bucket + a.count;
    *order_out = order;
    cudaError_t e = cudaMemsetAsync(hist, 0, sizeof(uint32_t) * kBuckets, st);
    if (e != cudaSuccess) return e;
    switch (family) {
        case TB_FAMILY_HS45: e = launch_key_fam<TB_FAMILY_HS45>(a, bucket, hist, st); break;
        case TB_FAMILY_BOXQP: e = launch_key_fam<TB_FAMILY_BOXQP>(a, bucket, hist, st); break;
        case TB_FAMILY_NCVX: e = launch_key_fam<TB_FAMILY_NCVX>(a, bucket, hist, st); break;
        case TB_FAMILY_BRANCH: e = launch_key_fam<TB_FAMILY_BRANCH>(a, bucket, hist, st); break;
        default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    order_scan_kernel<<<1, kScanThreads, 0, st>>>(hist, offs);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    order_scatter_kernel<<<(unsigned)((a.count + 255) / 256), 256, 0, st>>>(bucket, offs, order, a.count);
    note_launches(3);
    return cudaGetLastError();
}

}  // namespace tbdev
