// H2D bandwidth from a cudaHostAlloc(Portable) staging buffer right after a
// multi-threaded host copy into it (the library's pageable-input path).
// nvcc -O3 -arch=sm_100a h2d_staging.cu -o h2d_staging
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <cuda_runtime.h>
#include <emmintrin.h>

// copy with non-temporal stores (the staging is not left dirty in the CPU caches)
static void nt_copy(char* dst, const char* src, size_t n) {
    size_t i = 0;
    for (; i + 64 <= n; i += 64) {
        __m128i a = _mm_loadu_si128((const __m128i*)(src + i)), b = _mm_loadu_si128((const __m128i*)(src + i + 16)),
                c = _mm_loadu_si128((const __m128i*)(src + i + 32)), e = _mm_loadu_si128((const __m128i*)(src + i + 48));
        _mm_stream_si128((__m128i*)(dst + i), a); _mm_stream_si128((__m128i*)(dst + i + 16), b);
        _mm_stream_si128((__m128i*)(dst + i + 32), c); _mm_stream_si128((__m128i*)(dst + i + 48), e);
    }
    _mm_sfence();
    if (i < n) memcpy(dst + i, src + i, n - i);
}
int main() {
    const size_t parts[4] = {3145728, 3145728, 3145728, 18874368};
    size_t total = 0;
    for (size_t p : parts) total += p;
    std::vector<char> src(total, 1);
    char* h = nullptr;
    char* d = nullptr;
    cudaHostAlloc((void**)&h, total, cudaHostAllocPortable);
    cudaMalloc((void**)&d, total);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    for (int mode = 0; mode < 5; ++mode) {
        for (int r = 0; r < 5; ++r) {
            auto t0 = std::chrono::steady_clock::now();
            if (mode >= 1) {  // host copy into the staging, 8 threads (modes 3, 4: non-temporal stores)
                auto cp = [&](size_t k) {
                    const size_t a = total * k / 8, b = total * (k + 1) / 8;
                    if (mode >= 3) nt_copy(h + a, &src[a], b - a); else memcpy(h + a, &src[a], b - a);
                };
                std::vector<std::thread> th;
                for (int k = 1; k < 8; ++k) th.emplace_back(cp, k);
                cp(0);
                for (auto& x : th) x.join();
            }
            auto t1 = std::chrono::steady_clock::now();
            size_t off = 0;
            if (mode == 2 || mode == 4) {
                cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice, st);
            } else {
                for (size_t p : parts) { cudaMemcpyAsync(d + off, h + off, p, cudaMemcpyHostToDevice, st); off += p; }
            }
            cudaStreamSynchronize(st);
            auto t2 = std::chrono::steady_clock::now();
            auto ms = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count() * 1e3; };
            printf("mode %d: host copy %.3f ms, H2D %.3f ms (%.1f GB/s)\n", mode, ms(t0, t1), ms(t1, t2), total / ms(t1, t2) / 1e6);
        }
    }
}
