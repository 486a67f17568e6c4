// tronbatch_gpu/solve_batch.hpp — C++ drop-in for tronbatch::solve_batch
// (reference batch.hpp:27-78) on B200 GPUs, header-only over the C ABI
// (include/tb_capi.h, libtronbatch_b200.so).
//
// It reuses the reference's own types (tronbatch::TronConfig tron.hpp:54,
// SolveStatus :83, SolveReport :94, BatchResult batch.hpp:17, exceptions
// dense.hpp:15-24 / tron.hpp:21-24), so switching a caller is one line:
//
//     auto br = tronbatch::solve_batch(problems, x0s, cfg, workers);        // CPU reference
//     auto br = tronbatch::gpu::solve_batch(problems, x0s, cfg, {0, 1});   // B200s
//
// Problems must be device families (host callbacks cannot run on the GPU):
// the problem types below satisfy the reference BoundedProblem concept
// (tron.hpp:28-36) with host evaluations AND carry the family id + packed
// parameters the device evaluates with identical arithmetic.  Any type with
//     static constexpr int32_t family;  std::vector<double> params() const;
// plus dim()/lower()/upper() works.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "tronbatch/batch.hpp"
#include "tronbatch/tron.hpp"

#include "../tb_capi.h"
#include "../../paper_2106_14995_b200/csrc/tb_families.h"

namespace tronbatch::gpu {

// ------------------------------------------------------------- families
template <int32_t FAM>
struct FamilyProblem {
    static constexpr int32_t family = FAM;
    int n = 0;
    Vector l, u, prm;
    int dim() const { return n; }
    const Vector& lower() const { return l; }
    const Vector& upper() const { return u; }
    const Vector& params() const { return prm; }
    double eval_f(const Vector& x) const { return tb_family_f(FAM, x.data(), prm.data(), n); }
    Vector eval_grad(const Vector& x) const {
        Vector g(n);
        tb_family_grad(FAM, x.data(), prm.data(), n, g.data());
        return g;
    }
    DenseMatrix eval_hess(const Vector& x) const {
        DenseMatrix a(n);
        tb_family_hess(FAM, x.data(), prm.data(), n, a.data());
        return a;
    }
};

using NcvxProblem = FamilyProblem<TB_FAMILY_NCVX>;      // SURVEY §8(d) nonconvex family
using BranchProblem = FamilyProblem<TB_FAMILY_BRANCH>;  // ADMM branch subproblem, dim 4 / 6

// make_quadratic (tests/support/boxqp_oracle.hpp:44-62) as a device family
inline FamilyProblem<TB_FAMILY_BOXQP> make_quadratic(const DenseMatrix& h, const Vector& c, Vector l, Vector u) {
    FamilyProblem<TB_FAMILY_BOXQP> p;
    p.n = h.dim();
    p.l = std::move(l);
    p.u = std::move(u);
    p.prm.assign(h.data(), h.data() + std::size_t(p.n) * p.n);
    p.prm.insert(p.prm.end(), c.begin(), c.end());
    return p;
}

// Hs45Problem (batch.hpp:116-173) as a device family
inline FamilyProblem<TB_FAMILY_HS45> make_hs45(int n, int capacity = kDefaultCapacity) {
    Hs45Problem ref(n, capacity);  // same capacity check / exception
    FamilyProblem<TB_FAMILY_HS45> p;
    p.n = n;
    p.l = ref.lower();
    p.u = ref.upper();
    return p;
}

namespace detail {
// f(begin, end) over contiguous ranges of [0, n) on up to hardware_concurrency
// host threads (one thread below 8,192 items)
template <typename F>
void parallel_ranges(int64_t n, F&& f) {
    const int64_t hw = std::max<int64_t>(1, std::thread::hardware_concurrency());
    const int64_t t = std::min<int64_t>(hw, std::max<int64_t>(1, n / 8192));
    if (t <= 1) {
        f(int64_t(0), n);
        return;
    }
    std::vector<std::thread> pool;
    pool.reserve(t - 1);
    for (int64_t k = 1; k < t; ++k) pool.emplace_back([&, k] { f(n * k / t, n * (k + 1) / t); });
    f(int64_t(0), n / t);
    for (auto& th : pool) th.join();
}
}  // namespace detail

// ------------------------------------------------------------- context
class Context {
public:
    explicit Context(const std::vector<int>& devices = {0}) {
        std::vector<int32_t> d(devices.begin(), devices.end());
        tb_context* c = nullptr;
        if (tb_context_create(d.data(), static_cast<int32_t>(d.size()), &c) != TB_OK)
            throw std::runtime_error(std::string("tronbatch::gpu: ") + tb_last_error());
        ctx_.reset(c);
    }
    tb_context* get() const { return ctx_.get(); }

    // Page-locked pack / result buffers reused across calls (grown on demand):
    // the solve copies them straight into its pipeline (no staging, no page
    // faults of fresh allocations).  A Context is not thread-safe.
    struct Pinned {
        void* p = nullptr;
        size_t cap = 0;
        ~Pinned() { tb_host_free(p); }
        void* ensure(size_t bytes) {
            if (bytes <= cap) return p;
            tb_host_free(p);
            p = nullptr;
            cap = 0;
            if (tb_host_alloc(static_cast<int64_t>(bytes), &p) != TB_OK)
                throw std::runtime_error(std::string("tronbatch::gpu: ") + tb_last_error());
            cap = bytes;
            return p;
        }
    };
    Pinned& pack() const { return pack_; }
    Pinned& results() const { return results_; }

private:
    struct Del {
        void operator()(tb_context* c) const { tb_context_destroy(c); }
    };
    std::unique_ptr<tb_context, Del> ctx_;
    mutable Pinned pack_, results_;
};

inline tb_tron_config to_c(const TronConfig& cfg) {
    tb_tron_config c;
    tb_config_default(&c);
    c.tol_pg = cfg.tol_pg;
    c.has_delta0 = cfg.delta0.has_value() ? 1 : 0;
    c.delta0 = cfg.delta0.value_or(0.0);
    c.max_iter = cfg.max_iter;
    c.cg_tol = cfg.cg_tol;
    c.eta0 = cfg.eta0;
    c.sigma1 = cfg.sigma1;
    c.sigma2 = cfg.sigma2;
    c.sigma3 = cfg.sigma3;
    c.mu0 = cfg.mu0;
    c.mu1 = cfg.mu1;
    c.interp_factor = cfg.interp_factor;
    c.delta_max = cfg.delta_max;
    return c;
}

// solve_batch (batch.hpp:27-29): same arguments and result type; `devices`
// replaces `workers` (contiguous even partitions per device, batch.hpp:61-70).
// Throws exactly where the reference throws: invalid_argument for the config
// / lengths / dimensions / bounds, EvaluationError, SingularFactorError.
template <typename P>
BatchResult solve_batch(const std::vector<P>& problems, const std::vector<Vector>& x0s, const TronConfig& cfg,
                        const Context& ctx) {
    if (problems.size() != x0s.size()) throw std::invalid_argument("solve_batch: problems and x0s length mismatch");
    cfg.validate();
    BatchResult out;
    const int64_t N = static_cast<int64_t>(problems.size());
    if (N == 0) return out;
    const int n = problems[0].dim();
    const int64_t np = tb_family_nparams(P::family, n);
    if (np < 0) throw std::invalid_argument("solve_batch: dimension invalid for the problem family");
    for (int64_t i = 0; i < N; ++i) {
        const P& p = problems[i];
        if (p.dim() != n || static_cast<int>(x0s[i].size()) != n || static_cast<int>(p.lower().size()) != n ||
            static_cast<int>(p.upper().size()) != n)
            throw std::invalid_argument("solve: dimension mismatch");
    }
    // pack into the context's page-locked buffer (host threads like batch.hpp:61-70)
    const int64_t npk = std::max<int64_t>(np, 1);
    double* x0 = static_cast<double*>(ctx.pack().ensure(sizeof(double) * size_t(N) * size_t(3 * n + npk)));
    double *lo = x0 + N * n, *up = lo + N * n, *prm = up + N * n;
    detail::parallel_ranges(N, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i) {
            const P& p = problems[i];
            std::memcpy(&x0[i * n], x0s[i].data(), sizeof(double) * n);
            std::memcpy(&lo[i * n], p.lower().data(), sizeof(double) * n);
            std::memcpy(&up[i * n], p.upper().data(), sizeof(double) * n);
            if (np > 0) std::memcpy(&prm[i * np], p.params().data(), sizeof(double) * np);
        }
    });
    tb_problem_batch b{P::family, n, N, x0, lo, up, np > 0 ? prm : nullptr, np, TB_MEM_HOST};
    // results land in the context's page-locked buffer
    char* rb = static_cast<char*>(
        ctx.results().ensure(size_t(N) * (sizeof(double) * (n + 3) + sizeof(int32_t) * 2 + sizeof(int64_t) * 2)));
    double* xs = reinterpret_cast<double*>(rb);
    double *fs = xs + N * n, *pg = fs + N, *wt = pg + N;
    int64_t *cg = reinterpret_cast<int64_t*>(wt + N), *fe = cg + N;
    int32_t *st = reinterpret_cast<int32_t*>(fe + N), *it = st + N;
    tb_batch_result r{};
    r.x_star = xs;
    r.f_star = fs;
    r.pg_norm = pg;
    r.status = st;
    r.iterations = it;
    r.cg_iterations = cg;
    r.f_evals = fe;
    r.wall_time = wt;
    r.memspace = TB_MEM_HOST;
    const tb_tron_config c = to_c(cfg);
    const int rc = tb_solve_batch(ctx.get(), &b, &c, &r);
    if (rc == TB_E_INVALID_ARGUMENT) throw std::invalid_argument(tb_last_error());
    if (rc == TB_E_PROBLEM) {
        const std::string msg = tb_last_error();
        if (msg.find("EvaluationError") != std::string::npos) throw EvaluationError(msg);
        if (msg.find("SingularFactorError") != std::string::npos) throw SingularFactorError(msg);
        throw std::invalid_argument(msg);
    }
    if (rc != TB_OK) throw std::runtime_error(std::string("tronbatch::gpu: ") + tb_last_error());
    out.reports.resize(N);
    out.per_problem_time.assign(wt, wt + N);
    // one x_star vector per report (the reference's SolveReport): built by
    // host threads over contiguous ranges (per-thread malloc arenas)
    detail::parallel_ranges(N, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i) {
            SolveReport& s = out.reports[i];
            s.x_star.assign(&xs[i * n], &xs[i * n] + n);
            s.f_star = fs[i];
            s.pg_norm = pg[i];
            s.status = static_cast<SolveStatus>(st[i]);
            s.iterations = it[i];
            s.cg_iterations = cg[i];
            s.f_evals = fe[i];
            s.wall_time = wt[i];
        }
    });
    out.partition_times.assign(r.partition_times, r.partition_times + r.n_partitions);
    out.batch_wall_time = r.batch_wall_time;
    return out;
}

template <typename P>
BatchResult solve_batch(const std::vector<P>& problems, const std::vector<Vector>& x0s, const TronConfig& cfg = {},
                        const std::vector<int>& devices = {0}) {
    if (devices.empty()) throw std::invalid_argument("solve_batch: workers must be >= 1");
    Context ctx(devices);
    return solve_batch(problems, x0s, cfg, ctx);
}

}  // namespace tronbatch::gpu
