// tron_kernels.cu — family dispatch of the TRON kernels.
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>

#include "tb_families.h"
#include "tron_launch.h"
#include "tron_kernels.cuh"

namespace tbdev {
cudaError_t launch_hs45(const KernelArgs& a, cudaStream_t st);
cudaError_t launch_boxqp(const KernelArgs& a, cudaStream_t st);
cudaError_t launch_ncvx(const KernelArgs& a, cudaStream_t st);
cudaError_t launch_branch(const KernelArgs& a, cudaStream_t st);
cudaError_t ws_need_hs45(int n, long long count, int form, size_t* bytes);
cudaError_t ws_need_boxqp(int n, long long count, int form, size_t* bytes);
cudaError_t ws_need_ncvx(int n, long long count, int form, size_t* bytes);

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
cudaError_t tron_ws_need(int family, int n, long long count, int form, size_t* bytes) {
    *bytes = 0;
    if (count <= 0) return cudaSuccess;
    switch (family) {
        case TB_FAMILY_HS45: return ws_need_hs45(n, count, form, bytes);
        case TB_FAMILY_BOXQP: return ws_need_boxqp(n, count, form, bytes);
        case TB_FAMILY_NCVX: return ws_need_ncvx(n, count, form, bytes);
    }
    return cudaSuccess;
}

static std::atomic<long long> g_kernel_launches{0};
void note_launches(long long k) { g_kernel_launches += k; }
long long launches() { return g_kernel_launches.load(); }

// Counter slots: kSlots per device, handed out round-robin.  A slot is reused
// only after kSlots later persistent launches on the device, so concurrent
// launches (chunk streams, async callers) never share one.
namespace {
constexpr int kSlots = 4096;
std::mutex g_slot_mu;
unsigned long long* g_slots[64] = {};
unsigned g_slot_next[64] = {};
}  // namespace
cudaError_t counter_slot(unsigned long long** out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(g_slot_mu);
    if (!g_slots[dev]) {
        void* p = nullptr;
        if ((e = cudaMalloc(&p, sizeof(unsigned long long) * kSlots)) != cudaSuccess) return e;
        if ((e = cudaMemset(p, 0, sizeof(unsigned long long) * kSlots)) != cudaSuccess) return e;
        g_slots[dev] = static_cast<unsigned long long*>(p);
    }
    *out = g_slots[dev] + (g_slot_next[dev]++ % kSlots);
    return cudaSuccess;
}

int tron_form(int family, const KernelArgs& a) { return resolve_form(family, a); }
int device_sm_count() { return device_sms(); }

int max_warp_dim() { return 32; }
int max_dim() { return 128; }
}  // namespace tbdev
