// Latency microbenchmark (single warp, dependent chains) for the ops on the
// TRON kernel's critical path.  nvcc -arch=sm_100a --fmad=false -O3 latency.cu -o latency
#include <cstdio>
#include <cuda_runtime.h>
#define N 1024
__global__ void k(double* out, long long* cyc, double a, double b, int mode) {
    __shared__ double sm[64];
    double x = a + threadIdx.x * 1e-9, y = b;
    unsigned u = threadIdx.x;
    sm[threadIdx.x] = x;
    __syncwarp();
    long long t0 = clock64();
    switch (mode) {
        case 0: for (int i = 0; i < N; ++i) x = x + y; break;                       // DADD
        case 1: for (int i = 0; i < N; ++i) x = x * y; break;                       // DMUL
        case 2: for (int i = 0; i < N; ++i) x = fma(x, y, a); break;                // DFMA
        case 3: for (int i = 0; i < N; ++i) x = y / x; break;                       // IEEE div
        case 4: for (int i = 0; i < N; ++i) x = sqrt(x) + 1.0; break;               // sqrt+add
        case 5: for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31); break;
        case 6: for (int i = 0; i < N; ++i) { x = sm[(int)(x) & 31]; } break;       // LDS chain
        case 7: for (int i = 0; i < N; ++i) { u = __reduce_max_sync(0xffffffffu, u) + 1; } x = u; break;
        case 8: for (int i = 0; i < N; ++i) { sm[threadIdx.x] = x; __syncwarp(); x = sm[(threadIdx.x + 1) & 31] + 1.0; } break;
        case 9: for (int i = 0; i < N; ++i) { x = (x < y) ? y : x; x = x + 1e-300; } break;  // smax + add
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { *cyc = t1 - t0; }
    out[threadIdx.x] = x;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 64 * 8); cudaMalloc(&c, 8);
    const char* names[] = {"DADD", "DMUL", "DFMA", "DDIV(IEEE)", "DSQRT+DADD", "SHFL(64b)", "LDS(64b,dep)", "REDUX+IADD", "STS;WARPSYNC;LDS;DADD", "SEL-max+DADD"};
    for (int m = 0; m < 10; ++m) {
        long long h = 0;
        for (int r = 0; r < 3; ++r) { k<<<1, 32>>>(o, c, 1.0000001, 0.9999999, m); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); }
        printf("%-24s %6.1f cycles/op\n", names[m], (double)h / N);
    }
    return 0;
}
