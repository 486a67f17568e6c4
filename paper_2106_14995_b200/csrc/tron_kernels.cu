// tron_kernels.cu — family dispatch of the TRON kernels.
#include <cuda_runtime.h>

#include "tb_families.h"
#include "tron_launch.h"

namespace tbdev {
cudaError_t launch_hs45(const KernelArgs& a, cudaStream_t st);
cudaError_t launch_boxqp(const KernelArgs& a, cudaStream_t st);
cudaError_t launch_ncvx(const KernelArgs& a, cudaStream_t st);
cudaError_t launch_branch(const KernelArgs& a, cudaStream_t st);

cudaError_t launch_tron(int family, const KernelArgs& a, cudaStream_t st) {
    if (a.count <= 0) return cudaSuccess;
    switch (family) {
        case TB_FAMILY_HS45: return launch_hs45(a, st);
        case TB_FAMILY_BOXQP: return launch_boxqp(a, st);
        case TB_FAMILY_NCVX: return launch_ncvx(a, st);
        case TB_FAMILY_BRANCH: return launch_branch(a, st);
    }
    return cudaErrorInvalidValue;
}

int max_warp_dim() { return 32; }
}  // namespace tbdev
