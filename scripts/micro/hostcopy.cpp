// Host memcpy bandwidth with T threads (pageable -> page-locked-sized buffers):
// g++ -O3 -pthread hostcopy.cpp -o hostcopy && ./hostcopy
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
int main() {
    const size_t bytes = 28311552;
    std::vector<char> src(bytes, 1), dst(bytes, 0);
    for (int t : {1, 2, 4, 8, 16}) {
        double best = 1e9;
        for (int r = 0; r < 7; ++r) {
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> th;
            for (int k = 1; k < t; ++k)
                th.emplace_back([&, k] { std::memcpy(&dst[bytes * k / t], &src[bytes * k / t], bytes * (k + 1) / t - bytes * k / t); });
            std::memcpy(&dst[0], &src[0], bytes / t);
            for (auto& x : th) x.join();
            best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        }
        std::printf("%2d threads: %.3f ms = %.1f GB/s\n", t, best * 1e3, bytes / best / 1e9);
    }
}
