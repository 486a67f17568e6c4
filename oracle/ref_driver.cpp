// ref_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// Compiles the UNMODIFIED reference headers (/root/reference/proj/include/
// tronbatch/*.hpp and tests/support/*.hpp, included from where they lie) into
// oracle/_ref/libtronref.so with a small C ABI so Python tests and bench.py's
// cpu_baseline can run the reference's own solve_batch and primitives on the
// same buffers as the GPU.  No reference source is copied into this repo.
//
// Problem types handed to the reference templates:
//   HS45   -> tronbatch::Hs45Problem (batch.hpp:116), the reference's own
//   BOXQP  -> testutil::make_quadratic (tests/support/boxqp_oracle.hpp:44)
//   NCVX / BRANCH -> TwinProblem below: satisfies tronbatch::BoundedProblem
//             (tron.hpp:28-36) by evaluating csrc/tb_families.h
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "support/boxqp_oracle.hpp"
#include "support/test_util.hpp"
#include "tronbatch/batch.hpp"
#include "tronbatch/dense.hpp"
#include "tronbatch/tron.hpp"

#include "../include/tb_capi.h"
#include "../paper_2106_14995_b200/csrc/tb_families.h"

using namespace tronbatch;

namespace {

struct TwinProblem {
    int fam = 0, n = 0;
    Vector l, u;
    const double* prm = nullptr;
    int dim() const { return n; }
    const Vector& lower() const { return l; }
    const Vector& upper() const { return u; }
    double eval_f(const Vector& x) const { return tb_family_f(fam, x.data(), prm, n); }
    Vector eval_grad(const Vector& x) const {
        Vector g(n);
        tb_family_grad(fam, x.data(), prm, n, g.data());
        return g;
    }
    DenseMatrix eval_hess(const Vector& x) const {
        DenseMatrix a(n);
        tb_family_hess(fam, x.data(), prm, n, a.data());
        return a;
    }
};
static_assert(BoundedProblem<TwinProblem>);

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

TronConfig to_cfg(const tb_tron_config* c) {
    TronConfig cfg;
    cfg.tol_pg = c->tol_pg;
    if (c->has_delta0) cfg.delta0 = c->delta0;
    cfg.max_iter = c->max_iter;
    cfg.cg_tol = c->cg_tol;
    cfg.eta0 = c->eta0;
    cfg.sigma1 = c->sigma1;
    cfg.sigma2 = c->sigma2;
    cfg.sigma3 = c->sigma3;
    cfg.mu0 = c->mu0;
    cfg.mu1 = c->mu1;
    cfg.interp_factor = c->interp_factor;
    cfg.delta_max = c->delta_max;
    return cfg;
}

DenseMatrix to_mat(int n, const double* a) {
    DenseMatrix m(n);
    std::memcpy(m.data(), a, sizeof(double) * n * n);
    return m;
}

Vector to_vec(int n, const double* a) { return Vector(a, a + n); }

template <typename P>
int run_batch(const std::vector<P>& probs, const std::vector<Vector>& x0s, const TronConfig& cfg,
              int workers, int n, double* x_star, double* f_star, double* pg, int32_t* status,
              int32_t* iters, int64_t* cg, int64_t* fev, double* ppt, double* part_times,
              double* wall) {
    BatchResult br = solve_batch(probs, x0s, cfg, workers);
    for (size_t i = 0; i < br.reports.size(); ++i) {
        const SolveReport& r = br.reports[i];
        if (x_star) std::memcpy(x_star + i * n, r.x_star.data(), sizeof(double) * n);
        if (f_star) f_star[i] = r.f_star;
        if (pg) pg[i] = r.pg_norm;
        if (status) status[i] = static_cast<int32_t>(r.status);
        if (iters) iters[i] = r.iterations;
        if (cg) cg[i] = r.cg_iterations;
        if (fev) fev[i] = r.f_evals;
        if (ppt) ppt[i] = br.per_problem_time[i];
    }
    if (part_times)
        for (size_t k = 0; k < br.partition_times.size(); ++k) part_times[k] = br.partition_times[k];
    if (wall) *wall = br.batch_wall_time;
    return 0;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// solve_batch (batch.hpp:27-78) on the reference code.  Returns 0, or the
// TB_STATUS_* code of the exception the reference threw (3 EvaluationError,
// 4 invalid_argument, 5 SingularFactorError), message in ref_last_error().
int ref_solve_batch(int family, int n, int64_t count, const double* x0, const double* lower,
                    const double* upper, const double* params, int64_t stride,
                    const tb_tron_config* c, int workers, double* x_star, double* f_star,
                    double* pg, int32_t* status, int32_t* iters, int64_t* cg, int64_t* fev,
                    double* per_problem_time, double* partition_times, double* wall) {
    try {
        const TronConfig cfg = to_cfg(c);
        std::vector<Vector> x0s(count);
        for (int64_t i = 0; i < count; ++i) x0s[i] = to_vec(n, x0 + i * n);
        if (family == TB_FAMILY_HS45) {
            std::vector<Hs45Problem> probs;
            probs.reserve(count);
            for (int64_t i = 0; i < count; ++i) probs.push_back(make_hs45(n));
            return run_batch(probs, x0s, cfg, workers, n, x_star, f_star, pg, status, iters, cg,
                             fev, per_problem_time, partition_times, wall);
        }
        if (family == TB_FAMILY_BOXQP) {
            std::vector<FunctionProblem> probs;
            probs.reserve(count);
            for (int64_t i = 0; i < count; ++i) {
                const double* p = params + i * stride;
                probs.push_back(testutil::make_quadratic(to_mat(n, p), to_vec(n, p + n * n),
                                                         to_vec(n, lower + i * n),
                                                         to_vec(n, upper + i * n)));
            }
            return run_batch(probs, x0s, cfg, workers, n, x_star, f_star, pg, status, iters, cg,
                             fev, per_problem_time, partition_times, wall);
        }
        std::vector<TwinProblem> probs(count);
        for (int64_t i = 0; i < count; ++i) {
            probs[i].fam = family;
            probs[i].n = n;
            probs[i].l = to_vec(n, lower + i * n);
            probs[i].u = to_vec(n, upper + i * n);
            probs[i].prm = params + i * stride;
        }
        return run_batch(probs, x0s, cfg, workers, n, x_star, f_star, pg, status, iters, cg, fev,
                         per_problem_time, partition_times, wall);
    } catch (const EvaluationError& e) {
        return fail(e, TB_STATUS_EVALUATION_ERROR);
    } catch (const SingularFactorError& e) {
        return fail(e, TB_STATUS_SINGULAR_FACTOR);
    } catch (const std::invalid_argument& e) {
        return fail(e, TB_STATUS_ZERO_DIRECTION);
    } catch (const std::exception& e) {
        return fail(e, 99);
    }
}

// --- primitives (dense.hpp / tron.hpp), for primitive-level parity tests ---

double ref_dot(int n, const double* x, const double* y) { return dot(to_vec(n, x), to_vec(n, y)); }

void ref_gemv(int n, double alpha, const double* A, const double* x, double beta, const double* y,
              int transpose, double* out) {
    Vector r = gemv(alpha, to_mat(n, A), to_vec(n, x), beta, to_vec(n, y), transpose != 0);
    std::memcpy(out, r.data(), sizeof(double) * n);
}

int ref_ccf(int n, const double* A, int right, double* L, double* shift) {
    try {
        CholeskyResult c = right ? ccf_right_looking(to_mat(n, A)) : ccf(to_mat(n, A));
        std::memcpy(L, c.L.data(), sizeof(double) * n * n);
        *shift = c.shift;
        return 0;
    } catch (const FactorizationError& e) {
        return fail(e, TB_STATUS_FACTORIZATION_FAILED);
    }
}

int ref_trtrs(int n, const double* L, const double* b, int transpose, double* out) {
    try {
        Vector r = trtrs(to_mat(n, L), to_vec(n, b), transpose != 0);
        std::memcpy(out, r.data(), sizeof(double) * n);
        return 0;
    } catch (const SingularFactorError& e) {
        return fail(e, TB_STATUS_SINGULAR_FACTOR);
    }
}

double ref_pgnorm(int n, const double* x, const double* g, const double* l, const double* u) {
    return projected_gradient_norm(to_vec(n, x), to_vec(n, g), to_vec(n, l), to_vec(n, u));
}

void ref_gpstep(int n, const double* x, double alpha, const double* w, const double* l,
                const double* u, double* s) {
    Vector r = gpstep(to_vec(n, x), alpha, to_vec(n, w), to_vec(n, l), to_vec(n, u));
    std::memcpy(s, r.data(), sizeof(double) * n);
}

void ref_breakpt(int n, const double* x, const double* w, const double* l, const double* u,
                 int* count, double* bmin, double* bmax) {
    BreakpointInfo b = breakpt(to_vec(n, x), to_vec(n, w), to_vec(n, l), to_vec(n, u));
    *count = b.count;
    *bmin = b.min;
    *bmax = b.max;
}

int ref_trqsol(int n, const double* x, const double* w, double delta, double* sigma) {
    try {
        *sigma = trqsol(to_vec(n, x), to_vec(n, w), delta);
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, TB_STATUS_ZERO_DIRECTION);
    }
}

int ref_cauchy(int n, const double* x, const double* g, const double* A, const double* l,
               const double* u, double delta, const tb_tron_config* c, double alpha_start,
               double* alpha, double* s) {
    try {
        CauchyStep cs = cauchy(to_vec(n, x), to_vec(n, g), to_mat(n, A), to_vec(n, l), to_vec(n, u),
                               delta, to_cfg(c), alpha_start);
        *alpha = cs.alpha;
        std::memcpy(s, cs.s.data(), sizeof(double) * n);
        return 0;
    } catch (const EvaluationError& e) {
        return fail(e, TB_STATUS_EVALUATION_ERROR);
    }
}

int ref_precond_cg(int n, const double* A, const double* g, const double* L, double delta,
                   const tb_tron_config* c, double* step, int* status, int* iterations,
                   double* rel_residual) {
    try {
        CgResult r = precond_cg(to_mat(n, A), to_vec(n, g), to_mat(n, L), delta, to_cfg(c));
        std::memcpy(step, r.step.data(), sizeof(double) * n);
        *status = static_cast<int>(r.status);
        *iterations = r.iterations;
        *rel_residual = r.rel_residual;
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, TB_STATUS_ZERO_DIRECTION);
    }
}

void ref_line_search(int n, const double* x, const double* l, const double* u, const double* A,
                     const double* g, const double* w, const tb_tron_config* c, double* beta,
                     double* x_next) {
    LineSearchResult r = projected_line_search(to_vec(n, x), to_vec(n, l), to_vec(n, u),
                                               to_mat(n, A), to_vec(n, g), to_vec(n, w), to_cfg(c));
    *beta = r.beta;
    std::memcpy(x_next, r.x_next.data(), sizeof(double) * n);
}

int ref_imbalance(const double* times, int n_iters, int n_parts, double* nu, double* nu_max,
                  double* nu_min, double* nu_mean) {
    try {
        std::vector<std::vector<double>> t(n_iters, std::vector<double>(n_parts));
        for (int k = 0; k < n_iters; ++k)
            for (int p = 0; p < n_parts; ++p) t[k][p] = times[k * n_parts + p];
        ImbalanceStats s = imbalance(t);
        for (int k = 0; k < n_iters; ++k) nu[k] = s.nu_per_iter[k];
        *nu_max = s.nu_max;
        *nu_min = s.nu_min;
        *nu_mean = s.nu_mean;
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, TB_E_INVALID_ARGUMENT);
    }
}

int ref_config_validate(const tb_tron_config* c) {
    try {
        to_cfg(c).validate();
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, TB_E_INVALID_ARGUMENT);
    }
}

// The reference's own hs45 / make_quadratic evaluations, to pin the device
// family twins in tb_families.h bit-for-bit.
void ref_hs45_eval(int n, const double* x, double* f, double* g, double* H) {
    Hs45Problem p = make_hs45(n, 1 << 20);
    Vector xv = to_vec(n, x);
    *f = p.eval_f(xv);
    Vector gv = p.eval_grad(xv);
    std::memcpy(g, gv.data(), sizeof(double) * n);
    DenseMatrix h = p.eval_hess(xv);
    std::memcpy(H, h.data(), sizeof(double) * n * n);
}

void ref_boxqp_eval(int n, const double* Hq, const double* c, const double* x, double* f,
                    double* g) {
    FunctionProblem p = testutil::make_quadratic(to_mat(n, Hq), to_vec(n, c), Vector(n, -kInf),
                                                 Vector(n, kInf));
    Vector xv = to_vec(n, x);
    *f = p.eval_f(xv);
    Vector gv = p.eval_grad(xv);
    std::memcpy(g, gv.data(), sizeof(double) * n);
}

// testutil::boxqp_oracle (boxqp_oracle.hpp:67-139): brute-force active sets.
int ref_boxqp_oracle(int n, const double* Hq, const double* c, const double* l, const double* u,
                     double* x) {
    try {
        Vector r = testutil::boxqp_oracle(to_mat(n, Hq), to_vec(n, c), to_vec(n, l), to_vec(n, u));
        std::memcpy(x, r.data(), sizeof(double) * n);
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 99);
    }
}

}  // extern "C"
