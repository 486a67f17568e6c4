// dropin_trace.cpp -- timeline of the C++ drop-in on a C2 batch file (scripts/dropin_trace.py
// writes it): the solve_batch call vs destroying the previous BatchResult.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "tronbatch/batch.hpp"
#include "tronbatch_gpu/solve_batch.hpp"
using namespace tronbatch;
int main(int argc, char** argv) {
    std::FILE* f = std::fopen(argv[1], "rb");
    int64_t hdr[3];
    if (std::fread(hdr, sizeof hdr, 1, f) != 1) return 2;
    const int64_t N = hdr[0], n = hdr[1], np = hdr[2];
    std::vector<double> x0(N * n), lo(N * n), up(N * n), prm(N * np);
    if (std::fread(x0.data(), 8, x0.size(), f) != x0.size() || std::fread(lo.data(), 8, lo.size(), f) != lo.size() ||
        std::fread(up.data(), 8, up.size(), f) != up.size() || std::fread(prm.data(), 8, prm.size(), f) != prm.size()) return 2;
    std::vector<gpu::BranchProblem> problems(N);
    std::vector<Vector> x0s(N);
    for (int64_t i = 0; i < N; ++i) {
        problems[i].n = (int)n;
        problems[i].l.assign(&lo[i * n], &lo[i * n] + n);
        problems[i].u.assign(&up[i * n], &up[i * n] + n);
        problems[i].prm.assign(&prm[i * np], &prm[i * np] + np);
        x0s[i].assign(&x0[i * n], &x0[i * n] + n);
    }
    gpu::Context ctx({0});
    const TronConfig cfg{};
    for (int r = 0; r < 8; ++r) {
        auto t0 = std::chrono::steady_clock::now();
        BatchResult br = gpu::solve_batch(problems, x0s, cfg, ctx);
        auto t1 = std::chrono::steady_clock::now();
        { BatchResult gone = std::move(br); }
        auto t2 = std::chrono::steady_clock::now();
        std::printf("call %.3f ms (library wall %.3f ms), destroy result %.3f ms\n",
                    std::chrono::duration<double>(t1 - t0).count() * 1e3, br.batch_wall_time * 1e3,
                    std::chrono::duration<double>(t2 - t1).count() * 1e3);
    }
}
