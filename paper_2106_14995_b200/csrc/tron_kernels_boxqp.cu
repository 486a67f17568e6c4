// tron_kernels_boxqp.cu — TB_FAMILY_BOXQP kernels: D = next of {4, 8, 16, 32} >= dim.
#include "tron_kernels.cuh"

namespace tbdev {
cudaError_t launch_boxqp(const KernelArgs& a, cudaStream_t st) {
    if (a.n <= 4) return launch_fd<TB_FAMILY_BOXQP, 4>(a, st);
    if (a.n <= 8) return launch_fd<TB_FAMILY_BOXQP, 8>(a, st);
    if (a.n <= 16) return launch_fd<TB_FAMILY_BOXQP, 16>(a, st);
    return launch_fd<TB_FAMILY_BOXQP, 32>(a, st);
}
}  // namespace tbdev
