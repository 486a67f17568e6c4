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
// the TB_FORM_* launch_tron resolves `a` to (never TB_FORM_AUTO)
int tron_form(int family, const KernelArgs& a);
int max_dim();
cudaError_t tron_ws_need(int family, int n, long long count, int form, size_t* bytes);
// kernels of this library launched so far (TRON phases, ADMM stages)
void note_launches(long long k);
// a problem-counter slot on the current device for one persistent launch
// (round-robin over a pool; the launcher zeroes it on its stream)
cudaError_t counter_slot(unsigned long long** out);
long long launches();
// longest-expected-first launch order (tron_order.cu) into `ws`
// (order_ws_bytes(a.count) bytes); *order_out points into ws
size_t order_ws_bytes(long long count);
int device_sm_count();
cudaError_t launch_order(int family, const KernelArgs& a, void* ws, cudaStream_t st, const uint32_t** order_out);
}  // namespace tbdev
