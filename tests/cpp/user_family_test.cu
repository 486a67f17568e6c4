// user_family_test.cu — a caller-defined problem family (not one of the
// library's compiled-in families) through include/tronbatch_gpu/user_family.cuh:
// the same __host__ __device__ functions feed the reference's own CPU
// solve_batch (batch.hpp:27-78, via UserProblem's BoundedProblem interface)
// and the GPU kernel instantiated in THIS translation unit.  Every
// SolveReport field must be bit-identical.  Built into oracle/_ref/ (it
// compiles reference headers) by `make -C oracle ref`; runs on a GPU box.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

#include "tronbatch/batch.hpp"
#include "tronbatch_gpu/user_family.cuh"

using namespace tronbatch;

// Shifted, scaled extended Rosenbrock with a bilinear coupling (nonconvex):
//   f = sum_{i<n-1} a_i (y_{i+1} - y_i^2)^2 + (1 - y_i)^2 + b * sum_i y_i y_{(i+1) mod n},
//   y = x - c.  params: c[n], a[n-1], b.
struct ShiftedRosen {
    static constexpr int kMaxDim = 16;
    __host__ __device__ static double y(const double* x, const double* p, int i) { return x[i] - p[i]; }
    __host__ __device__ static double f(const double* x, const double* p, int n) {
        const double* a = p + n;
        const double b = p[2 * n - 1];
        double s = 0.0;
        for (int i = 0; i + 1 < n; ++i) {
            const double yi = y(x, p, i), yj = y(x, p, i + 1);
            const double r = yj - yi * yi, q = 1.0 - yi;
            s += a[i] * (r * r) + q * q;
        }
        for (int i = 0; i < n; ++i) s += b * (y(x, p, i) * y(x, p, (i + 1) % n));
        return s;
    }
    __host__ __device__ static double grad(const double* x, const double* p, int n, int i) {
        const double* a = p + n;
        const double b = p[2 * n - 1];
        const double yi = y(x, p, i);
        double g = 0.0;
        if (i + 1 < n) {
            const double r = y(x, p, i + 1) - yi * yi;
            g += a[i] * (2.0 * r) * (-2.0 * yi) - 2.0 * (1.0 - yi);
        }
        if (i > 0) {
            const double ym = y(x, p, i - 1);
            g += a[i - 1] * (2.0 * (yi - ym * ym));
        }
        g += b * (y(x, p, (i + 1) % n) + y(x, p, (i + n - 1) % n));
        return g;
    }
    __host__ __device__ static double hess(const double* x, const double* p, int n, int i, int j) {
        const double* a = p + n;
        const double b = p[2 * n - 1];
        double h = 0.0;
        if (i == j) {
            const double yi = y(x, p, i);
            if (i + 1 < n) h += a[i] * (12.0 * yi * yi - 4.0 * y(x, p, i + 1)) + 2.0;
            if (i > 0) h += 2.0 * a[i - 1];
        } else {
            const int lo = i < j ? i : j, hi = i < j ? j : i;
            if (hi == lo + 1) h += -4.0 * a[lo] * y(x, p, lo);
        }
        if (n > 2 && ((i + 1) % n == j || (j + 1) % n == i)) h += b;
        if (n == 2 && i != j) h += 2.0 * b;
        if (n == 1) h += 2.0 * b;
        return h;
    }
};

static bool same_bits(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0 || (a != a && b != b); }

int main() {
    std::mt19937_64 rng(20260);
    std::uniform_real_distribution<double> U(-1.0, 1.0);
    int fails = 0, total = 0;
    for (int n : {1, 2, 3, 5, 8, 13, 16}) {
        std::vector<gpu::UserProblem<ShiftedRosen>> probs;
        std::vector<Vector> x0s;
        for (int k = 0; k < 300; ++k) {
            gpu::UserProblem<ShiftedRosen> p;
            p.n = n;
            p.l.resize(n);
            p.u.resize(n);
            p.prm.resize(2 * n);
            for (int i = 0; i < n; ++i) {
                p.prm[i] = 0.5 * U(rng);                       // c
                p.l[i] = -1.5 + 0.5 * U(rng);
                p.u[i] = 1.5 + 0.5 * U(rng);
            }
            for (int i = 0; i + 1 < n; ++i) p.prm[n + i] = 5.0 + 45.0 * (0.5 + 0.5 * U(rng));  // a
            p.prm[2 * n - 1] = 0.3 * U(rng);                    // b (coupling, may make it indefinite)
            Vector x0(n);
            for (int i = 0; i < n; ++i) x0[i] = 1.2 * U(rng);
            probs.push_back(p);
            x0s.push_back(x0);
        }
        const BatchResult cpu = solve_batch(probs, x0s, TronConfig{}, 4);  // the reference, unmodified
        const BatchResult gpu = gpu::solve_batch_user(probs, x0s, TronConfig{});
        int bad = 0, conv = 0;
        for (size_t i = 0; i < probs.size(); ++i) {
            const SolveReport &a = gpu.reports[i], &b = cpu.reports[i];
            bool ok = a.status == b.status && a.iterations == b.iterations && a.cg_iterations == b.cg_iterations &&
                      a.f_evals == b.f_evals && same_bits(a.f_star, b.f_star) && same_bits(a.pg_norm, b.pg_norm);
            for (int k = 0; k < n; ++k) ok = ok && same_bits(a.x_star[k], b.x_star[k]);
            bad += !ok;
            conv += b.status == SolveStatus::Converged;
        }
        std::printf("user family ShiftedRosen n=%2d: %zu problems, %d converged (reference), %d differ\n", n,
                    probs.size(), conv, bad);
        fails += bad;
        total += (int)probs.size();
    }
    std::printf("%s: %d of %d problems differ\n", fails ? "FAIL" : "PASS", fails, total);
    return fails ? 1 : 0;
}
