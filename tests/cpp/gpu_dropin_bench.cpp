// gpu_dropin_bench.cpp — end-to-end time of the C++ drop-in
// (include/tronbatch_gpu/solve_batch.hpp) on a batch written by bench.py:
// std::vector<BranchProblem> + std::vector<Vector> x0s in, BatchResult out,
// exactly what a reference caller switching from tronbatch::solve_batch
// (batch.hpp:27-78) gets.  The timed call includes the drop-in's packing of
// the problems into the ABI arrays, the library's pinned staging of those
// pageable arrays, the chunked H2D / solve / D2H pipeline, and the
// construction of the 65,536 SolveReports.
// usage: gpu_dropin_bench <batch.bin> [reps]   (prints one JSON line)
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tronbatch/batch.hpp"
#include "tronbatch_gpu/solve_batch.hpp"

using namespace tronbatch;

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s batch.bin [reps]\n", argv[0]);
        return 2;
    }
    const int reps = argc > 2 ? std::atoi(argv[2]) : 7;
    std::FILE* f = std::fopen(argv[1], "rb");
    if (!f) return 2;
    int64_t hdr[3];  // N, n, np
    if (std::fread(hdr, sizeof hdr, 1, f) != 1) return 2;
    const int64_t N = hdr[0], n = hdr[1], np = hdr[2];
    std::vector<double> x0(N * n), lo(N * n), up(N * n), prm(N * np);
    bool ok = std::fread(x0.data(), sizeof(double), x0.size(), f) == x0.size() &&
              std::fread(lo.data(), sizeof(double), lo.size(), f) == lo.size() &&
              std::fread(up.data(), sizeof(double), up.size(), f) == up.size() &&
              std::fread(prm.data(), sizeof(double), prm.size(), f) == prm.size();
    std::fclose(f);
    if (!ok) return 2;
    std::vector<gpu::BranchProblem> problems(N);
    std::vector<Vector> x0s(N);
    for (int64_t i = 0; i < N; ++i) {
        gpu::BranchProblem& p = problems[i];
        p.n = static_cast<int>(n);
        p.l.assign(&lo[i * n], &lo[i * n] + n);
        p.u.assign(&up[i * n], &up[i * n] + n);
        p.prm.assign(&prm[i * np], &prm[i * np] + np);
        x0s[i].assign(&x0[i * n], &x0[i * n] + n);
    }
    gpu::Context ctx({0});
    const TronConfig cfg{};
    BatchResult br;
    for (int w = 0; w < 2; ++w) br = gpu::solve_batch(problems, x0s, cfg, ctx);
    std::vector<double> t;
    std::vector<double> t_with_free;  // the same call plus destroying the previous BatchResult
    for (int k = 0; k < reps; ++k) {
        const auto t0 = std::chrono::steady_clock::now();
        br = gpu::solve_batch(problems, x0s, cfg, ctx);
        t_with_free.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    for (int k = 0; k < reps; ++k) {
        br = BatchResult{};  // the previous result's 65,536 vectors are freed before the clock starts
        const auto t0 = std::chrono::steady_clock::now();
        BatchResult r = gpu::solve_batch(problems, x0s, cfg, ctx);
        t.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        br = std::move(r);
    }
    std::sort(t.begin(), t.end());
    std::sort(t_with_free.begin(), t_with_free.end());
    const double med = t[t.size() / 2];
    const double med_free = t_with_free[t_with_free.size() / 2];
    long conv = 0;
    for (const auto& r : br.reports) conv += r.status == SolveStatus::Converged;
    std::printf("{\"value\": %.6g, \"unit\": \"solves/s\", \"median_s\": %.6g, \"best_s\": %.6g, \"reps\": %d, "
                "\"problems\": %lld, \"converged\": %ld, \"batch_wall_time\": %.6g, "
                "\"value_incl_freeing_previous_result\": %.6g}\n",
                N / med, med, t[0], reps, (long long)N, conv, br.batch_wall_time, N / med_free);
    return 0;
}
