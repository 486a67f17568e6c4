// Does a warp interleave two divergent dependent chains (ITS), or serialize?
#include <cstdio>
#include <cuda_runtime.h>
#define N 4096
__global__ void k(double* out, long long* cyc, double a, int mode) {
    double x = a + threadIdx.x * 1e-9;
    long long t0 = clock64();
    if (mode == 0) {                       // all lanes: one chain
        for (int i = 0; i < N; ++i) x = x * a + 1e-300;
    } else if (mode == 1) {                // two halves take different branches, same length
        if (threadIdx.x < 16) { for (int i = 0; i < N; ++i) x = x * a + 1e-300; }
        else { for (int i = 0; i < N; ++i) x = x * a - 1e-300; }
    } else if (mode == 2) {                // same but with data-dependent loop bounds
        int n = N + (threadIdx.x < 16 ? 0 : 1);
        if (threadIdx.x < 16) { for (int i = 0; i < n; ++i) x = x * a + 1e-300; }
        else { for (int i = 0; i < n; ++i) x = x * a - 1e-300; }
    } else {                               // 4 groups
        int g = threadIdx.x / 8;
        if (g == 0) { for (int i = 0; i < N; ++i) x = x * a + 1e-300; }
        else if (g == 1) { for (int i = 0; i < N; ++i) x = x * a - 1e-300; }
        else if (g == 2) { for (int i = 0; i < N; ++i) x = x * a + 2e-300; }
        else { for (int i = 0; i < N; ++i) x = x * a - 2e-300; }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) *cyc = t1 - t0;
    out[threadIdx.x] = x;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 32 * 8); cudaMalloc(&c, 8);
    const char* nm[] = {"uniform chain", "2 divergent halves", "2 divergent (dyn bounds)", "4 divergent groups"};
    for (int m = 0; m < 4; ++m) {
        long long h = 0;
        for (int r = 0; r < 3; ++r) { k<<<1, 32>>>(o, c, 0.9999999, m); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); }
        printf("%-28s %8.1f cycles/iter\n", nm[m], (double)h / N);
    }
}
