// tron_kernels.cu — instantiation and launch dispatch of the TRON kernels.
#include <cuda_runtime.h>

#include "tron_device.cuh"
#include "tron_launch.h"

namespace tbdev {

template <int FAM, int D>
static cudaError_t launch_fd(const KernelArgs& a, cudaStream_t st) {
    const int np = (a.nparams + 1) & ~1;
    const size_t smem = sizeof(double) * (size_t)(SmemLayout<D>::fixed() + np);
    auto kern = tron_solve_kernel<FAM, D>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    kern<<<(unsigned)a.count, 32, smem, st>>>(a);
    return cudaGetLastError();
}

template <int FAM>
static cudaError_t launch_f(const KernelArgs& a, cudaStream_t st) {
    if (a.n <= 4) return launch_fd<FAM, 4>(a, st);
    if (FAM == TB_FAMILY_BRANCH) return launch_fd<FAM, 8>(a, st);
    if (a.n <= 8) return launch_fd<FAM, 8>(a, st);
    if (a.n <= 16) return launch_fd<FAM, 16>(a, st);
    return launch_fd<FAM, 32>(a, st);
}

cudaError_t launch_tron(int family, const KernelArgs& a, cudaStream_t st) {
    if (a.count <= 0) return cudaSuccess;
    switch (family) {
        case TB_FAMILY_HS45: return launch_f<TB_FAMILY_HS45>(a, st);
        case TB_FAMILY_BOXQP: return launch_f<TB_FAMILY_BOXQP>(a, st);
        case TB_FAMILY_NCVX: return launch_f<TB_FAMILY_NCVX>(a, st);
        case TB_FAMILY_BRANCH: return launch_f<TB_FAMILY_BRANCH>(a, st);
    }
    return cudaErrorInvalidValue;
}

int max_warp_dim() { return 32; }

}  // namespace tbdev
