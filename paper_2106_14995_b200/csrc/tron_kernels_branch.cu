// tron_kernels_branch.cu — ADMM branch family kernels, D = dim exactly (4, 6).
#include "tron_kernels.cuh"
#include "tron_thread.cuh"

namespace tbdev {
cudaError_t launch_branch(const KernelArgs& a, cudaStream_t st) {
    if (thread_form(a, 4096)) return launch_thread<4, TB_FAMILY_BRANCH>(a, st);
    if (a.n == 4) return launch_fd<TB_FAMILY_BRANCH, 4>(a, st);
    return launch_fd<TB_FAMILY_BRANCH, 6>(a, st);
}
}  // namespace tbdev

#ifdef TB_PHASES
// debug build only: per-phase cycle totals of this family's kernels
extern "C" int tb_debug_read_phases_branch(unsigned long long* out) {
    if (cudaMemcpyFromSymbol(out, tbdev::g_phase_cycles, sizeof(unsigned long long) * 16) != cudaSuccess) return 2;
    unsigned long long z[16] = {};
    return cudaMemcpyToSymbol(tbdev::g_phase_cycles, z, sizeof z) == cudaSuccess ? 0 : 2;
}
#endif
