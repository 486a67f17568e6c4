// tron_kernels_branch.cu — ADMM branch family kernels, D = dim exactly (4, 6).
#include "tron_kernels.cuh"

namespace tbdev {
// D = dim exactly (4 or 6): thread form (n = 4, large batches) or warp form
cudaError_t launch_branch(const KernelArgs& a, cudaStream_t st) {
    switch (resolve_form(TB_FAMILY_BRANCH, a)) {
        case TB_FORM_THREAD: return launch_thread<4, TB_FAMILY_BRANCH>(a, st);
    }
    return a.n == 4 ? launch_fd<TB_FAMILY_BRANCH, 4>(a, st) : launch_fd<TB_FAMILY_BRANCH, 6>(a, st);
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
