// tron_kernels.cuh — instantiation and launch of the TRON kernels for one
// family (one translation unit per family: parallel builds, smaller objects).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "tron_block.cuh"
#include "tron_device.cuh"
#include "tron_launch.h"

namespace tbdev {

template <int FAM, int D, bool COUNT>
static cudaError_t launch_fdc(const KernelArgs& a, cudaStream_t st) {
    const int np = (a.nparams + 1) & ~1;
    const size_t smem = sizeof(double) * (size_t)(SmemLayout<D>::fixed() + np);
    auto kern = tron_solve_kernel<FAM, D, COUNT>;
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

// ---------------------------------------------------------------- d > 32
// Hessian placement of the block kernel: TB_BLOCK_ASMEM=1 keeps A in shared
// memory (fewer resident problems per SM), default 0 keeps it in the
// L2-resident global workspace.
inline bool blk_asmem() {
    const char* e = std::getenv("TB_BLOCK_ASMEM");
    return e && e[0] == '1';
}

// Dimension routing (ncvx, B = 32,768, device-resident, ms):
//   d        12     16     17..20        24     32
//   warp    8.65  11.41  24.4 / 27.4     -      -     (D = 16 / 32 warp kernel)
//   blk32  10.96  14.47  ~/ 20.19      25.98  48.21   (one-warp block kernel)
//   blk64  14.85  19.28  ~/ 25.22      30.19  50.10
// so d <= 16 runs the warp kernel, 17..32 the one-warp D = 32 block kernel
// (compacted systems, 8/16-lane lockstep attempt groups), 33..64 D = 64 and
// 65..128 D = 128.  TB_BLOCK_MIN_DIM (9..33) and TB_BLOCK32=0 override.
inline int blk_min_dim() {
    const char* e = std::getenv("TB_BLOCK_MIN_DIM");
    const int v = e ? std::atoi(e) : 17;
    return v < 9 ? 9 : v;
}
inline bool blk32() {
    const char* e = std::getenv("TB_BLOCK32");
    return !(e && e[0] == '0');
}

// persistent grid: resident blocks per SM x SMs, capped by the batch
template <int FAM, int D, bool ASMEM, bool COUNT>
static cudaError_t blk_grid(long long count, long long* grid, size_t* smem_out) {
    using SL = BlkLayout<D, ASMEM>;
    const size_t smem = sizeof(double) * (size_t)SL::total();
    auto kern = tron_block_kernel<FAM, D, ASMEM, COUNT>;
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

template <int FAM, int D, bool ASMEM, bool COUNT>
static cudaError_t launch_blk_c(const KernelArgs& a, cudaStream_t st) {
    long long grid = 0;
    size_t smem = 0;
    cudaError_t e = blk_grid<FAM, D, ASMEM, COUNT>(a.count, &grid, &smem);
    if (e != cudaSuccess) return e;
    using SL = BlkLayout<D, ASMEM>;
    const size_t need = kBlkWsHeader + (ASMEM ? 0 : sizeof(double) * (size_t)grid * D * D) +
                        (SL::LP < SL::LPFULL ? sizeof(double) * (size_t)grid * SL::LPFULL : 0);
    if (!a.ws || a.ws_bytes < need) return cudaErrorMemoryAllocation;
    if ((e = cudaMemsetAsync(a.ws, 0, sizeof(unsigned), st)) != cudaSuccess) return e;
    tron_block_kernel<FAM, D, ASMEM, COUNT><<<(unsigned)grid, D, smem, st>>>(a);
    note_launches(1);
    return cudaGetLastError();
}

template <int FAM, int D>
static cudaError_t launch_blk(const KernelArgs& a, cudaStream_t st) {
    if (blk_asmem())
        return a.flops ? launch_blk_c<FAM, D, true, true>(a, st) : launch_blk_c<FAM, D, true, false>(a, st);
    return a.flops ? launch_blk_c<FAM, D, false, true>(a, st) : launch_blk_c<FAM, D, false, false>(a, st);
}

// workspace bytes the block kernel needs for `count` problems of dim n
template <int FAM, int D>
static cudaError_t ws_need_blk(long long count, size_t* bytes) {
    long long grid = 0;
    size_t smem = 0;
    *bytes = kBlkWsHeader;
    const bool as = blk_asmem();
    cudaError_t e = as ? blk_grid<FAM, D, true, false>(count, &grid, &smem)
                       : blk_grid<FAM, D, false, false>(count, &grid, &smem);
    if (e != cudaSuccess) return e;
    long long g2 = 0;
    if ((e = as ? blk_grid<FAM, D, true, true>(count, &g2, &smem) : blk_grid<FAM, D, false, true>(count, &g2, &smem)) !=
        cudaSuccess)
        return e;
    if (g2 > grid) grid = g2;
    using SL = BlkLayout<D, false>;
    if (!as) *bytes += sizeof(double) * (size_t)grid * D * D;
    if (SL::LP < SL::LPFULL) *bytes += sizeof(double) * (size_t)grid * SL::LPFULL;
    return cudaSuccess;
}

}  // namespace tbdev
