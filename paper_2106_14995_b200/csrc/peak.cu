// peak.cu — FP64 (non-tensor) DFMA throughput microbenchmark, the roofline
// denominator for the TRON kernel (MEASURED_PEAKS.json has HBM and bf16 only).
// Many independent DFMA chains per thread, grid = 8 x SMs blocks of 256.
#include <cuda_runtime.h>

#include "../../include/tb_capi.h"

namespace {
constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void __launch_bounds__(256) dfma_kernel(double* out, double a, double b) {
    double acc[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = threadIdx.x * 1e-3 + c;
#pragma unroll 1
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += acc[c];
    if (s == 1234.5) out[0] = s;  // keep the work alive
}
}  // namespace

// Measures DFMA throughput on `device`; writes TFLOP/s (FMA = 2 flops).
extern "C" int tb_measure_fp64_peak(int32_t device, double* tflops) {
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) return TB_E_CUDA;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    double* out = nullptr;
    cudaMalloc(&out, sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8;
    dfma_kernel<<<blocks, 256>>>(out, 0.999999, 1e-9);  // warm-up
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) dfma_kernel<<<blocks, 256>>>(out, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * kChains * (double)kIters * blocks * 256.0 * reps;
    *tflops = flops / (ms * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    cudaSetDevice(prev);
    return err == cudaSuccess ? TB_OK : TB_E_CUDA;
}
