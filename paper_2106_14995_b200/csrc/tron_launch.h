// tron_launch.h — internal interface between the C ABI layer and the kernels.
#pragma once
#include <cuda_runtime.h>

namespace tbdev {
struct KernelArgs;
}
#include "tron_device.cuh"
namespace tbdev {
cudaError_t launch_tron(int family, const KernelArgs& a, cudaStream_t st);
int max_warp_dim();
int max_dim();
cudaError_t tron_ws_need(int family, int n, long long count, size_t* bytes);
// kernels of this library launched so far (TRON phases, ADMM stages)
void note_launches(long long k);
long long launches();
}  // namespace tbdev
