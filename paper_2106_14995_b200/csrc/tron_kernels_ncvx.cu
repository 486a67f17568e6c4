// tron_kernels_ncvx.cu — TB_FAMILY_NCVX kernels: D = next of {4, 8, 16, 32} >= dim (one warp per
// problem) up to d = 16; above it the block kernel with D = 32, 64 or 128 threads (tron_kernels.cuh).
#include "tron_kernels.cuh"
#include "tron_thread.cuh"

namespace tbdev {
cudaError_t launch_ncvx(const KernelArgs& a, cudaStream_t st) {
    if (thread_form(a, 16384)) return launch_thread<4, TB_FAMILY_NCVX>(a, st);
    if (a.n <= 4) return launch_fd<TB_FAMILY_NCVX, 4>(a, st);
    if (a.n <= 8) return launch_fd<TB_FAMILY_NCVX, 8>(a, st);
    if (a.n >= blk_min_dim()) {
        if (a.n <= 32 && blk32()) return launch_blk<TB_FAMILY_NCVX, 32>(a, st);
        if (a.n <= 64) return launch_blk<TB_FAMILY_NCVX, 64>(a, st);
        return launch_blk<TB_FAMILY_NCVX, 128>(a, st);
    }
    if (a.n <= 16) return launch_fd<TB_FAMILY_NCVX, 16>(a, st);
    return launch_fd<TB_FAMILY_NCVX, 32>(a, st);
}
cudaError_t ws_need_ncvx(int n, long long count, size_t* bytes) {
    *bytes = 0;
    if (n <= 8 || n < blk_min_dim()) return cudaSuccess;
    if (n <= 32 && blk32()) return ws_need_blk<TB_FAMILY_NCVX, 32>(count, bytes);
    if (n <= 64) return ws_need_blk<TB_FAMILY_NCVX, 64>(count, bytes);
    return ws_need_blk<TB_FAMILY_NCVX, 128>(count, bytes);
}
}  // namespace tbdev

#ifdef TB_PHASES
// debug build only: per-phase cycle totals of this family's kernels
extern "C" int tb_debug_read_phases_ncvx(unsigned long long* out) {
    if (cudaMemcpyFromSymbol(out, tbdev::g_phase_cycles, sizeof(unsigned long long) * 16) != cudaSuccess) return 2;
    unsigned long long z[16] = {};
    return cudaMemcpyToSymbol(tbdev::g_phase_cycles, z, sizeof z) == cudaSuccess ? 0 : 2;
}
#endif
