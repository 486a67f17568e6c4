// tron_kernels_hs45.cu — TB_FAMILY_HS45 kernels: D = next of {4, 8, 16, 32} >= dim.
#include "tron_kernels.cuh"

namespace tbdev {
cudaError_t launch_hs45(const KernelArgs& a, cudaStream_t st) {
    if (a.n <= 4) return launch_fd<TB_FAMILY_HS45, 4>(a, st);
    if (a.n <= 8) return launch_fd<TB_FAMILY_HS45, 8>(a, st);
    if (a.n <= 16) return launch_fd<TB_FAMILY_HS45, 16>(a, st);
    return launch_fd<TB_FAMILY_HS45, 32>(a, st);
}
}  // namespace tbdev
