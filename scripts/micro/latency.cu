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
        case 10: for (int i = 0; i < N; ++i) x = __drcp_rn(x) + 1.0; break;                 // RN reciprocal + add
        case 11: for (int i = 0; i < N; ++i) {                                             // Markstein a*RN(1/d)
            const double q0 = x * y, e = fma(-q0, a, x); x = fma(e, y, q0);
            const unsigned ex = ((unsigned)__double2hiint(x) >> 20) & 0x7FFu;
            if (ex - 64u > 1918u) x = x / a;
        } break;
        case 12: for (int i = 0; i < N; ++i) { const double d = sqrt(x); x = (y / d) + 1.0; } break;  // ccf: sqrt, div
        case 13: for (int i = 0; i < N; ++i) {                                             // ccf: sqrt, rcp, Markstein
            const double d = sqrt(x), r = __drcp_rn(d);
            const double q0 = y * r, e = fma(-q0, d, y); double q = fma(e, r, q0);
            const unsigned ex = ((unsigned)__double2hiint(q0) >> 20) & 0x7FFu;
            if (ex - 64u > 1918u) q = y / d;
            x = q + 1.0;
        } break;
        case 14: for (int i = 0; i < N; ++i) { const double d = sqrt(x); x = d * 0.5 + 1.0; } break;  // sqrt alone + mul + add
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { *cyc = t1 - t0; }
    out[threadIdx.x] = x;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 64 * 8); cudaMalloc(&c, 8);
    const char* names[] = {"DADD", "DMUL", "DFMA", "DDIV(IEEE)", "DSQRT+DADD", "SHFL(64b)", "LDS(64b,dep)", "REDUX+IADD", "STS;WARPSYNC;LDS;DADD", "SEL-max+DADD", "DRCP_RN+DADD", "Markstein(3 ops+guard)", "DSQRT->DDIV->DADD", "DSQRT->DRCP->Markstein->DADD", "DSQRT->DMUL->DADD"};
    for (int m = 0; m < 15; ++m) {
        long long h = 0;
        for (int r = 0; r < 3; ++r) { k<<<1, 32>>>(o, c, 1.0000001, 0.9999999, m); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); }
        printf("%-24s %6.1f cycles/op\n", names[m], (double)h / N);
    }
    return 0;
}
