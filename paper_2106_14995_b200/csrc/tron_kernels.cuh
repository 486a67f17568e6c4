// tron_kernels.cuh — instantiation and launch of the TRON kernels for one
// family (one translation unit per family: parallel builds, smaller objects).
#pragma once
#include <cuda_runtime.h>

#include "tron_device.cuh"

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
    return cudaGetLastError();
}

template <int FAM, int D>
static cudaError_t launch_fd(const KernelArgs& a, cudaStream_t st) {
    return a.flops ? launch_fdc<FAM, D, true>(a, st) : launch_fdc<FAM, D, false>(a, st);
}

}  // namespace tbdev
