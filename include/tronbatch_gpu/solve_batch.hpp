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
#include <condition_variable>
#include <cstdint>
#include <exception>
#include <functional>
#include <mutex>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#if defined(__SSE2__)
#include <emmintrin.h>
#endif

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
// Copy `count` doubles into the library's page-locked staging with streaming
// stores: a transfer of lines the CPU just wrote normally (dirty in its
// caches) runs at a third of the link rate (host buffers).
inline void stage_copy(double* dst, const double* src, std::size_t count) {
#if defined(__SSE2__)
    std::size_t i = 0;
    if (reinterpret_cast<std::uintptr_t>(dst) & 15) {
        dst[0] = src[0];
        i = 1;
    }
    for (; i + 2 <= count; i += 2) _mm_stream_pd(dst + i, _mm_loadu_pd(src + i));
    if (i < count) dst[i] = src[i];
#else
    std::memcpy(dst, src, sizeof(double) * count);
#endif
}

// A fixed pool of host threads owned by the Context: the drop-in packs and
// unpacks per pipeline chunk, and starting threads for every chunk would cost
// more than the copies they share.
class Pool {
public:
    explicit Pool(int n) : nt_(std::max(1, n)) {
        for (int k = 1; k < nt_; ++k) th_.emplace_back([this, k] { loop(k); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    Pool(const Pool&) = delete;
    Pool& operator=(const Pool&) = delete;

    // f(begin, end) over contiguous ranges of [0, n), at least `grain` items each
    template <typename F>
    void run(int64_t n, int64_t grain, F&& f) {
        const int64_t t = std::min<int64_t>(nt_, std::max<int64_t>(1, n / std::max<int64_t>(1, grain)));
        if (t <= 1) {
            if (n > 0) f(int64_t(0), n);
            return;
        }
        const std::function<void(int)> job = [&](int k) {
            if (k < t) f(n * k / t, n * (k + 1) / t);
        };
        {
            std::lock_guard<std::mutex> g(m_);
            job_ = &job;
            pending_ = nt_ - 1;
            ++gen_;
        }
        cv_.notify_all();
        job(0);
        std::unique_lock<std::mutex> l(m_);
        done_.wait(l, [&] { return pending_ == 0; });
        job_ = nullptr;
    }

private:
    void loop(int k) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(int)>* job;
            {
                std::unique_lock<std::mutex> l(m_);
                cv_.wait(l, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
                job = job_;
            }
            (*job)(k);
            std::lock_guard<std::mutex> g(m_);
            if (--pending_ == 0) done_.notify_one();
        }
    }
    int nt_;
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    const std::function<void(int)>* job_ = nullptr;
    uint64_t gen_ = 0;
    int pending_ = 0;
    bool stop_ = false;
};
}  // namespace detail

// ------------------------------------------------------------- context
class Context {
public:
    explicit Context(const std::vector<int>& devices = {0})
        : pool_(std::make_unique<detail::Pool>(static_cast<int>(std::thread::hardware_concurrency()))) {
        std::vector<int32_t> d(devices.begin(), devices.end());
        tb_context* c = nullptr;
        if (tb_context_create(d.data(), static_cast<int32_t>(d.size()), &c) != TB_OK)
            throw std::runtime_error(std::string("tronbatch::gpu: ") + tb_last_error());
        ctx_.reset(c);
    }
    tb_context* get() const { return ctx_.get(); }
    // host threads for packing / report building (a Context is not thread-safe)
    detail::Pool& pool() const { return *pool_; }

private:
    struct Del {
        void operator()(tb_context* c) const { tb_context_destroy(c); }
    };
    std::unique_ptr<tb_context, Del> ctx_;
    std::unique_ptr<detail::Pool> pool_;
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
    // The library pipelines the batch in chunks: it asks for each chunk's
    // inputs just before copying them to the device (pack) and hands over
    // each chunk's results as soon as they arrive (unpack), so packing the
    // problems and building the SolveReports (host threads, like
    // batch.hpp:61-70) overlap the device work on the other chunks.
    // The SolveReports (one heap vector each) are allocated on a helper
    // thread while the device works; the first unpack waits for it.
    out.per_problem_time.resize(N);
    std::exception_ptr prep_err;
    std::thread prep([&] {
        try {
            out.reports.resize(N);
            for (SolveReport& rep : out.reports) rep.x_star.resize(n);
        } catch (...) {
            prep_err = std::current_exception();
        }
    });
    struct Job {
        const std::vector<P>* problems;
        const std::vector<Vector>* x0s;
        BatchResult* out;
        detail::Pool* pool;
        std::thread* prep;
        std::exception_ptr* prep_err;
        int n;
        int64_t np;
        std::exception_ptr err;
    } job{&problems, &x0s, &out, &ctx.pool(), &prep, &prep_err, n, np, nullptr};
    constexpr int64_t kGrain = 1024;  // problems per host thread and range
    const tb_pack_fn pack = [](void* u, int64_t a, int64_t b, double* x0, double* lo, double* up, double* prm) {
        Job& j = *static_cast<Job*>(u);
        const int n = j.n;
        const int64_t np = j.np;
        j.pool->run(b - a, kGrain, [&](int64_t s, int64_t e) {
            for (int64_t i = s; i < e; ++i) {
                const P& p = (*j.problems)[a + i];
                detail::stage_copy(&x0[i * n], (*j.x0s)[a + i].data(), n);
                detail::stage_copy(&lo[i * n], p.lower().data(), n);
                detail::stage_copy(&up[i * n], p.upper().data(), n);
                if (np > 0) detail::stage_copy(&prm[i * np], p.params().data(), np);
            }
#if defined(__SSE2__)
            _mm_sfence();
#endif
        });
    };
    const tb_unpack_fn unpack = [](void* u, int64_t a, int64_t b, const tb_batch_result* r) {
        Job& j = *static_cast<Job*>(u);
        if (j.prep->joinable()) j.prep->join();
        if (*j.prep_err) return;  // rethrown after the call
        const int n = j.n;
        j.pool->run(b - a, kGrain, [&](int64_t s, int64_t e) {
            try {
                for (int64_t i = s; i < e; ++i) {
                    SolveReport& rep = j.out->reports[a + i];
                    std::memcpy(rep.x_star.data(), &r->x_star[i * n], sizeof(double) * n);
                    rep.f_star = r->f_star[i];
                    rep.pg_norm = r->pg_norm[i];
                    rep.status = static_cast<SolveStatus>(r->status[i]);
                    rep.iterations = r->iterations[i];
                    rep.cg_iterations = r->cg_iterations[i];
                    rep.f_evals = r->f_evals[i];
                    rep.wall_time = r->wall_time[i];
                    j.out->per_problem_time[a + i] = r->wall_time[i];
                }
            } catch (...) {  // (bad_alloc) never across the C ABI; rethrown below
                static std::mutex m;
                std::lock_guard<std::mutex> g(m);
                if (!j.err) j.err = std::current_exception();
            }
        });
    };
    tb_batch_result r{};
    const tb_tron_config c = to_c(cfg);
    const int rc = tb_solve_batch_packed(ctx.get(), P::family, n, N, &c, pack, unpack, &job, &r);
    if (prep.joinable()) prep.join();  // an error before any unpack
    if (prep_err) std::rethrow_exception(prep_err);
    if (job.err) std::rethrow_exception(job.err);
    if (rc == TB_E_INVALID_ARGUMENT) throw std::invalid_argument(tb_last_error());
    if (rc == TB_E_PROBLEM) {
        const std::string msg = tb_last_error();
        if (msg.find("EvaluationError") != std::string::npos) throw EvaluationError(msg);
        if (msg.find("SingularFactorError") != std::string::npos) throw SingularFactorError(msg);
        throw std::invalid_argument(msg);
    }
    if (rc != TB_OK) throw std::runtime_error(std::string("tronbatch::gpu: ") + tb_last_error());
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
