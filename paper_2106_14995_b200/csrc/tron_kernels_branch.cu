// tron_kernels_branch.cu — ADMM branch family kernels, D = dim exactly (4, 6).
#include "tron_kernels.cuh"

namespace tbdev {
cudaError_t launch_branch(const KernelArgs& a, cudaStream_t st) {
    if (a.n == 4) return launch_fd<TB_FAMILY_BRANCH, 4>(a, st);
    return launch_fd<TB_FAMILY_BRANCH, 6>(a, st);
}
}  // namespace tbdev
