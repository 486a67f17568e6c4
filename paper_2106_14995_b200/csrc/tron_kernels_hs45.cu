// tron_kernels_hs45.cu — TB_FAMILY_HS45 kernels: D = next of {4, 8, 16, 32} >= dim (one warp per
// problem) up to d = 16; above it the block kernel (tron_kernels.cuh).
#include "tron_kernels.cuh"

namespace tbdev {
cudaError_t launch_hs45(const KernelArgs& a, cudaStream_t st) { return launch_family<TB_FAMILY_HS45>(a, st); }
cudaError_t ws_need_hs45(int n, long long count, int form, size_t* bytes) {
    return family_ws_need<TB_FAMILY_HS45>(n, count, form, bytes);
}
}  // namespace tbdev

#ifdef TB_PHASES
// debug build only: per-phase cycle totals of this family's kernels
extern "C" int tb_debug_read_phases_hs45(unsigned long long* out) {
    if (cudaMemcpyFromSymbol(out, tbdev::g_phase_cycles, sizeof(unsigned long long) * 16) != cudaSuccess) return 2;
    unsigned long long z[16] = {};
    return cudaMemcpyToSymbol(tbdev::g_phase_cycles, z, sizeof z) == cudaSuccess ? 0 : 2;
}
#endif
