// tron_kernels.cuh — instantiation and launch of the TRON kernels for one
// family (one translation unit per family: parallel builds, smaller objects).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "tron_block.cuh"
#include "tron_device.cuh"
#include "tron_launch.h"
#include "tron_thread.cuh"

namespace tbdev {

// SMs of the current device (cached per device)
inline int device_sms() {
    static int sms[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (!sms[dev]) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v < 1) v = 148;
        sms[dev] = v;
    }
    return sms[dev];
}

#ifndef TB_ORD_MINB
#define TB_ORD_MINB 0  // experiments: resident blocks per SM of the ranked warp kernel (0: WarpMinBlocks<D>)
#endif

template <int FAM, int D, bool COUNT>
static cudaError_t launch_fdc(const KernelArgs& a, cudaStream_t st) {
    const int np = (a.nparams + 1) & ~1;
    const size_t smem = sizeof(double) * (size_t)(SmemLayout<D>::fixed() + np);
    auto kern = tron_solve_kernel<FAM, D, COUNT>;
    // the latency variant for batches (the whole partition, not a pipeline
    // chunk) that fit kLatencyBlocks warps per SM; counting runs are untimed
    if constexpr (!COUNT && WarpMinBlocks<D>::value > kLatencyBlocks) {
        const long long total = a.route_count > a.count ? a.route_count : a.count;
        if (total <= (long long)kLatencyBlocks * device_sms()) kern = tron_solve_kernel<FAM, D, false, kLatencyBlocks>;
    }
    // ranked launch (tron_order.cu; never a counting run)
    if constexpr (!COUNT)
        if (a.order) kern = tron_solve_kernel<FAM, D, false, TB_ORD_MINB ? TB_ORD_MINB : WarpMinBlocks<D>::value, true>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    kern<<<(unsigned)a.count, 32, smem, st>>>(a);
    note_launches(1);
    return cudaGetLastError();
}

template <int FAM, int D>
static cudaError_t launch_fd(const KernelArgs& a, cudaStream_t st) {
    return a.flops ? launch_fdc<FAM, D, true>(a, st) : launch_fdc<FAM, D, false>(a, st);
}

// ---------------------------------------------------------------- d > 16
// Hessian placement of the block kernel: compile with -DTB_BLOCK_ASMEM=1 to
// keep A in shared memory (fewer resident problems per SM; experiments), the
// default keeps it in the L2-resident global workspace.
#ifndef TB_BLOCK_ASMEM
#define TB_BLOCK_ASMEM 0
#endif

// Dimension routing (ncvx, B = 32,768, device-resident, ms):
//   d        12     16     17..20        24     32
//   warp    8.65  11.41  24.4 / 27.4     -      -     (D = 16 / 32 warp kernel)
//   blk32  10.96  14.47  ~/ 20.19      25.98  48.21   (one-warp block kernel)
//   blk64  14.85  19.28  ~/ 25.22      30.19  50.10
// so d <= 16 runs the warp kernel, 17..32 the one-warp D = 32 block kernel
// (compacted systems, 8/16-lane lockstep attempt groups), 33..64 D = 64 and
// 65..128 D = 128.  TB_FORM_WARP keeps d = 17..32 on the D = 32 warp kernel,
// TB_FORM_BLOCK moves d = 9..16 to the block kernel.
inline bool use_block(int n, int form) {
    if (n >= 17) return !(form == TB_FORM_WARP && n <= 32);
    return form == TB_FORM_BLOCK && n >= 9;
}
inline int block_dim(int n) { return n <= 32 ? 32 : (n <= 64 ? 64 : 128); }

// persistent grid: resident blocks per SM x SMs, capped by the batch
template <int FAM, int D, bool ASMEM, bool COUNT, bool ORD = false>
static cudaError_t blk_grid(long long count, long long* grid, size_t* smem_out) {
    using SL = BlkLayout<D, ASMEM>;
    const size_t smem = sizeof(double) * (size_t)SL::total();
    auto kern = tron_block_kernel<FAM, D, ASMEM, COUNT, ORD>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, D, smem)) != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    *grid = count < (long long)sms * per_sm ? count : (long long)sms * per_sm;
    *smem_out = smem;
    return cudaSuccess;
}

template <int FAM, int D, bool ASMEM, bool COUNT, bool ORD = false>
static cudaError_t launch_blk_c(const KernelArgs& a, cudaStream_t st) {
    if constexpr (!COUNT && !ORD)
        if (a.order) return launch_blk_c<FAM, D, ASMEM, false, true>(a, st);  // ranked work items
    long long grid = 0;
    size_t smem = 0;
    cudaError_t e = blk_grid<FAM, D, ASMEM, COUNT, ORD>(a.count, &grid, &smem);
    if (e != cudaSuccess) return e;
    using SL = BlkLayout<D, ASMEM>;
    const size_t need = kBlkWsHeader + (ASMEM ? 0 : sizeof(double) * (size_t)grid * D * D) +
                        (SL::LP < SL::LPFULL ? sizeof(double) * (size_t)grid * SL::LPFULL : 0);
    if (!a.ws || a.ws_bytes < need) return cudaErrorMemoryAllocation;
    if ((e = cudaMemsetAsync(a.ws, 0, sizeof(unsigned), st)) != cudaSuccess) return e;
    tron_block_kernel<FAM, D, ASMEM, COUNT, ORD><<<(unsigned)grid, D, smem, st>>>(a);
    note_launches(1);
    return cudaGetLastError();
}

template <int FAM, int D>
static cudaError_t launch_blk(const KernelArgs& a, cudaStream_t st) {
    constexpr bool AS = TB_BLOCK_ASMEM != 0;
    return a.flops ? launch_blk_c<FAM, D, AS, true>(a, st) : launch_blk_c<FAM, D, AS, false>(a, st);
}

// workspace bytes the block kernel needs for `count` problems of dim n
template <int FAM, int D>
static cudaError_t ws_need_blk(long long count, size_t* bytes) {
    long long grid = 0;
    size_t smem = 0;
    *bytes = kBlkWsHeader;
    constexpr bool as = TB_BLOCK_ASMEM != 0;
    cudaError_t e = blk_grid<FAM, D, as, false>(count, &grid, &smem);
    if (e != cudaSuccess) return e;
    long long g2 = 0;
    if ((e = blk_grid<FAM, D, as, true>(count, &g2, &smem)) != cudaSuccess) return e;
    if (g2 > grid) grid = g2;
    if ((e = blk_grid<FAM, D, as, false, true>(count, &g2, &smem)) != cudaSuccess) return e;  // ranked variant
    if (g2 > grid) grid = g2;
    using SL = BlkLayout<D, false>;
    if (!as) *bytes += sizeof(double) * (size_t)grid * D * D;
    if (SL::LP < SL::LPFULL) *bytes += sizeof(double) * (size_t)grid * SL::LPFULL;
    return cudaSuccess;
}

// ---------------------------------------------------------------- routing
// n = 4 without flop counting: TB_FORM_THREAD, or TB_FORM_AUTO on batches
// (the whole batch / partition, not the pipeline chunk) of >= min_count
inline bool thread_form(const KernelArgs& a, long long min_count) {
    if (a.flops || a.n != 4 || min_count < 0) return false;
    if (a.form == TB_FORM_THREAD) return true;
    if (a.form != TB_FORM_AUTO) return false;
    const long long total = a.route_count > a.count ? a.route_count : a.count;
    return total >= min_count;
}

// the one routing decision (launchers and tron_form): block kernel for large
// d, thread form for big n = 4 batches of the families that have it (branch
// from 4,096 problems, ncvx from 8,192), the warp kernel
// otherwise
inline int resolve_form(int family, const KernelArgs& a) {
    if (family != TB_FAMILY_BRANCH && use_block(a.n, a.form)) return TB_FORM_BLOCK;
    const long long min_thread = family == TB_FAMILY_BRANCH ? 4096 : (family == TB_FAMILY_NCVX ? 8192 : -1);
    if (thread_form(a, min_thread)) return TB_FORM_THREAD;
    return TB_FORM_WARP;
}

// hs45 / boxqp / ncvx: D = next of {4, 8, 16, 32} >= dim on the warp form,
// the block kernel above (use_block)
template <int FAM>
static cudaError_t launch_family(const KernelArgs& a, cudaStream_t st) {
    const int n = a.n;
    switch (resolve_form(FAM, a)) {
        case TB_FORM_BLOCK: {
            const int D = block_dim(n);
            if (D == 32) return launch_blk<FAM, 32>(a, st);
            if (D == 64) return launch_blk<FAM, 64>(a, st);
            return launch_blk<FAM, 128>(a, st);
        }
        case TB_FORM_THREAD:
            if constexpr (FAM == TB_FAMILY_NCVX) return launch_thread<4, FAM>(a, st);
            return cudaErrorInvalidValue;
    }
    if (n <= 4) return launch_fd<FAM, 4>(a, st);
    if (n <= 8) return launch_fd<FAM, 8>(a, st);
    if (n <= 16) return launch_fd<FAM, 16>(a, st);
    return launch_fd<FAM, 32>(a, st);
}

// workspace bytes the block kernel needs (0: another form)
template <int FAM>
static cudaError_t family_ws_need(int n, long long count, int form, size_t* bytes) {
    *bytes = 0;
    if (FAM == TB_FAMILY_BRANCH || !use_block(n, form)) return cudaSuccess;
    const int D = block_dim(n);
    if (D == 32) return ws_need_blk<FAM, 32>(count, bytes);
    if (D == 64) return ws_need_blk<FAM, 64>(count, bytes);
    return ws_need_blk<FAM, 128>(count, bytes);
}

}  // namespace tbdev
