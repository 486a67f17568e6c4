// tron_kernels_ncvx.cu — TB_FAMILY_NCVX kernels: D = next of {4, 8, 16, 32} >= dim.
#include "tron_kernels.cuh"

namespace tbdev {
cudaError_t launch_ncvx(const KernelArgs& a, cudaStream_t st) {
    if (a.n <= 4) return launch_fd<TB_FAMILY_NCVX, 4>(a, st);
    if (a.n <= 8) return launch_fd<TB_FAMILY_NCVX, 8>(a, st);
    if (a.n <= 16) return launch_fd<TB_FAMILY_NCVX, 16>(a, st);
    return launch_fd<TB_FAMILY_NCVX, 32>(a, st);
}
}  // namespace tbdev
