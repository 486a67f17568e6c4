// tron_kernels.cu — family dispatch of the TRON kernels.
#include <cuda_runtime.h>

#include <atomic>

#include "tb_families.h"
#include "tron_launch.h"

namespace tbdev {
cudaError_t launch_hs45(const KernelArgs& a, cudaStream_t st);
cudaError_t launch_boxqp(const KernelArgs& a, cudaStream_t st);
cudaError_t launch_ncvx(const KernelArgs& a, cudaStream_t st);
cudaError_t launch_branch(const KernelArgs& a, cudaStream_t st);
cudaError_t ws_need_hs45(int n, long long count, size_t* bytes);
cudaError_t ws_need_boxqp(int n, long long count, size_t* bytes);
cudaError_t ws_need_ncvx(int n, long long count, size_t* bytes);

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

// workspace bytes launch_tron needs in KernelArgs::ws (0 for the warp kernel)
cudaError_t tron_ws_need(int family, int n, long long count, size_t* bytes) {
    *bytes = 0;
    if (count <= 0) return cudaSuccess;
    switch (family) {
        case TB_FAMILY_HS45: return ws_need_hs45(n, count, bytes);
        case TB_FAMILY_BOXQP: return ws_need_boxqp(n, count, bytes);
        case TB_FAMILY_NCVX: return ws_need_ncvx(n, count, bytes);
    }
    return cudaSuccess;
}

static std::atomic<long long> g_kernel_launches{0};
void note_launches(long long k) { g_kernel_launches += k; }
long long launches() { return g_kernel_launches.load(); }

int max_warp_dim() { return 32; }
int max_dim() { return 128; }
}  // namespace tbdev
