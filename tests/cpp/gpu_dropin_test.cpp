// gpu_dropin_test.cpp — the C++ drop-in (include/tronbatch_gpu/solve_batch.hpp)
// against the reference's own CPU solve_batch, written like the reference's
// tests (tests/unit/tron_test.cpp): same problem factories (test_util.hpp,
// boxqp_oracle.hpp), same checks, plus bitwise equality of every report.
// Built into oracle/_ref/ (it compiles reference headers) by `make -C oracle ref`.
#include <cmath>
#include <cstdio>
#include <limits>
#include <string>

#include "support/boxqp_oracle.hpp"
#include "support/test_util.hpp"
#include "tronbatch/batch.hpp"
#include "tronbatch_gpu/solve_batch.hpp"

using namespace tronbatch;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                             \
    do {                                                                     \
        ++g_checks;                                                          \
        if (!(c)) {                                                          \
            ++g_fail;                                                        \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);          \
        }                                                                    \
    } while (0)

static bool same_bits(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0 || (a != a && b != b); }

static void same_reports(const BatchResult& g, const BatchResult& r, const char* what) {
    CHECK(g.reports.size() == r.reports.size());
    int bad = 0;
    for (size_t i = 0; i < r.reports.size(); ++i) {
        const SolveReport &a = g.reports[i], &b = r.reports[i];
        bool ok = a.status == b.status && a.iterations == b.iterations && a.cg_iterations == b.cg_iterations &&
                  a.f_evals == b.f_evals && same_bits(a.f_star, b.f_star) && same_bits(a.pg_norm, b.pg_norm);
        for (size_t k = 0; k < b.x_star.size(); ++k) ok = ok && same_bits(a.x_star[k], b.x_star[k]);
        bad += !ok;
    }
    std::printf("%-34s %zu problems, %d differ\n", what, r.reports.size(), bad);
    CHECK(bad == 0);
}

int main() {
    gpu::Context ctx({0});
    // tron_test.cpp:196-212: random 4-D box QPs vs the brute-force oracle
    {
        std::vector<gpu::FamilyProblem<TB_FAMILY_BOXQP>> gp;
        std::vector<FunctionProblem> rp;
        std::vector<Vector> x0s, expect;
        for (int t = 0; t < 50; ++t) {
            const int n = 4;
            const DenseMatrix h = testutil::random_spd(n, 0.5);
            Vector c = testutil::random_vector(n, -2.0, 2.0);
            Vector l(n), u(n);
            for (int i = 0; i < n; ++i) {
                l[i] = testutil::uniform(-1.0, 0.0);
                u[i] = l[i] + testutil::uniform(0.2, 1.5);
            }
            gp.push_back(gpu::make_quadratic(h, c, l, u));
            rp.push_back(testutil::make_quadratic(h, c, l, u));
            x0s.push_back(testutil::random_vector(n, -1.0, 1.0));
            expect.push_back(testutil::boxqp_oracle(h, c, l, u));
        }
        const BatchResult g = gpu::solve_batch(gp, x0s, TronConfig{}, ctx);
        const BatchResult r = solve_batch(rp, x0s, TronConfig{}, 4);
        same_reports(g, r, "box QPs (tron_test.cpp:196)");
        for (size_t i = 0; i < expect.size(); ++i) {
            CHECK(g.reports[i].status == SolveStatus::Converged);
            CHECK(testutil::max_abs_diff(g.reports[i].x_star, expect[i]) <= 1e-6);
        }
    }
    // tron_test.cpp:185-194 and SPEC acceptance 1: hs45 family
    {
        std::vector<gpu::FamilyProblem<TB_FAMILY_HS45>> gp;
        std::vector<Hs45Problem> rp;
        std::vector<Vector> x0s;
        for (int n = 1; n <= 32; ++n) {
            gp.push_back(gpu::make_hs45(n));
            rp.push_back(make_hs45(n));
            x0s.push_back(rp.back().default_start());
        }
        // one call per dimension (a batch has one dimension)
        for (int n = 1; n <= 32; ++n) {
            const BatchResult g = gpu::solve_batch(std::vector{gp[n - 1]}, std::vector<Vector>{x0s[n - 1]}, TronConfig{}, ctx);
            const BatchResult r = solve_batch(std::vector{rp[n - 1]}, std::vector<Vector>{x0s[n - 1]});
            if (n == 3 || n == 32) same_reports(g, r, ("hs45 n=" + std::to_string(n)).c_str());
            CHECK(g.reports[0].status == SolveStatus::Converged);
            for (int i = 0; i < n; ++i) CHECK(std::fabs(g.reports[0].x_star[i] - (i + 1)) <= 1e-6);
        }
    }
    // block-kernel sizes (d > 20): indefinite box QPs at d = 24 / 48 / 100 and
    // hs45 up to the reference's capacity (batch.hpp:15, 64), bitwise
    for (int n : {24, 48, 100}) {
        std::vector<gpu::FamilyProblem<TB_FAMILY_BOXQP>> gp;
        std::vector<FunctionProblem> rp;
        std::vector<Vector> x0s;
        for (int t = 0; t < (n > 64 ? 6 : 24); ++t) {
            DenseMatrix h(n);
            for (int j = 0; j < n; ++j)
                for (int i = j; i < n; ++i) h(i, j) = h(j, i) = testutil::uniform(-1.0, 1.0);
            Vector c = testutil::random_vector(n, -1.5, 1.5);
            Vector l(n), u(n);
            for (int i = 0; i < n; ++i) {
                l[i] = testutil::uniform(-1.5, -0.5);
                u[i] = testutil::uniform(0.5, 1.5);
            }
            gp.push_back(gpu::make_quadratic(h, c, l, u));
            rp.push_back(testutil::make_quadratic(h, c, l, u));
            x0s.push_back(testutil::random_vector(n, -0.5, 0.5));
        }
        const BatchResult g = gpu::solve_batch(gp, x0s, TronConfig{}, ctx);
        const BatchResult r = solve_batch(rp, x0s, TronConfig{}, 4);
        same_reports(g, r, ("indefinite box QPs d=" + std::to_string(n)).c_str());
    }
    for (int n : {33, 64}) {
        const BatchResult g = gpu::solve_batch(std::vector{gpu::make_hs45(n)},
                                               std::vector<Vector>{make_hs45(n).default_start()}, TronConfig{}, ctx);
        const BatchResult r = solve_batch(std::vector{make_hs45(n)}, std::vector<Vector>{make_hs45(n).default_start()});
        same_reports(g, r, ("hs45 n=" + std::to_string(n)).c_str());
    }
    // tron_test.cpp:251-266: NaN Hessian surfaces as FactorizationFailed
    {
        DenseMatrix h(2);
        h(0, 0) = 1.0;
        h(1, 1) = std::numeric_limits<double>::quiet_NaN();
        auto gp = std::vector{gpu::make_quadratic(h, Vector{0.0, 0.5}, Vector{-1, -1}, Vector{1, 1})};
        const BatchResult g = gpu::solve_batch(gp, std::vector<Vector>{{0.5, 0.5}}, TronConfig{}, ctx);
        CHECK(g.reports[0].status == SolveStatus::FactorizationFailed);
    }
    // tron_test.cpp:268-278: config validation throws std::invalid_argument
    {
        TronConfig bad;
        bad.sigma2 = 1.5;
        bool threw = false;
        try {
            gpu::solve_batch(std::vector{gpu::make_hs45(3)}, std::vector<Vector>{{0.5, 0.5, 0.5}}, bad, ctx);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    }
    // EvaluationError propagates out of solve_batch (tron.hpp:192, batch.hpp:75-76)
    {
        DenseMatrix h = DenseMatrix::identity(3);
        h(0, 0) = std::numeric_limits<double>::infinity();
        auto gp = std::vector{gpu::make_quadratic(h, Vector{0.1, 0.2, 0.3}, Vector(3, -1.0), Vector(3, 1.0))};
        bool threw = false;
        try {
            gpu::solve_batch(gp, std::vector<Vector>{{0.5, 0.5, 0.5}}, TronConfig{}, ctx);
        } catch (const EvaluationError&) {
            threw = true;
        }
        auto rp = std::vector{testutil::make_quadratic(h, Vector{0.1, 0.2, 0.3}, Vector(3, -1.0), Vector(3, 1.0))};
        bool ref_threw = false;
        try {
            solve_batch(rp, std::vector<Vector>{{0.5, 0.5, 0.5}});
        } catch (const EvaluationError&) {
            ref_threw = true;
        }
        CHECK(threw == ref_threw);
    }
    std::printf("{\"checks\": %d, \"failed\": %d}\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
