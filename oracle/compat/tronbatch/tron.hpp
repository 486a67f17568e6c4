// oracle/compat/tronbatch/tron.hpp — TEST INFRASTRUCTURE ONLY.
// The reference's tron.hpp API over the plain-C oracle (see dense.hpp here).
#pragma once
#include <concepts>
#include <functional>
#include <limits>
#include <optional>

#include "tronbatch/dense.hpp"

namespace tronbatch {

inline constexpr double kInf = std::numeric_limits<double>::infinity();

class EvaluationError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

template <typename P>
concept BoundedProblem = requires(const P& p, const Vector& x) {
    { p.dim() } -> std::convertible_to<int>;
    { p.lower() } -> std::convertible_to<Vector>;
    { p.upper() } -> std::convertible_to<Vector>;
    { p.eval_f(x) } -> std::convertible_to<double>;
    { p.eval_grad(x) } -> std::convertible_to<Vector>;
    { p.eval_hess(x) } -> std::convertible_to<DenseMatrix>;
};

struct FunctionProblem {
    int n = 0;
    Vector l, u;
    std::function<double(const Vector&)> f;
    std::function<Vector(const Vector&)> grad;
    std::function<DenseMatrix(const Vector&)> hess;
    int dim() const { return n; }
    const Vector& lower() const { return l; }
    const Vector& upper() const { return u; }
    double eval_f(const Vector& x) const { return f(x); }
    Vector eval_grad(const Vector& x) const { return grad(x); }
    DenseMatrix eval_hess(const Vector& x) const { return hess(x); }
};

struct TronConfig {
    double tol_pg = 1e-6;
    std::optional<double> delta0;
    int max_iter = 200;
    double cg_tol = 0.1;
    double eta0 = 1e-4;
    double sigma1 = 0.25;
    double sigma2 = 0.5;
    double sigma3 = 4.0;
    double mu0 = 1e-2;
    double mu1 = 1.0;
    double interp_factor = 0.5;
    double delta_max = 1e10;

    tb_tron_config c() const {
        tb_tron_config r;
        orc_config_default(&r);
        r.tol_pg = tol_pg;
        r.has_delta0 = delta0.has_value();
        r.delta0 = delta0.value_or(0.0);
        r.max_iter = max_iter;
        r.cg_tol = cg_tol;
        r.eta0 = eta0;
        r.sigma1 = sigma1;
        r.sigma2 = sigma2;
        r.sigma3 = sigma3;
        r.mu0 = mu0;
        r.mu1 = mu1;
        r.interp_factor = interp_factor;
        r.delta_max = delta_max;
        return r;
    }
    void validate() const {
        const tb_tron_config r = c();
        const char* msg;
        if (orc_config_validate(&r, &msg)) throw std::invalid_argument(msg);
    }
};

enum class SolveStatus { Converged, IterLimit, FactorizationFailed };

struct SolveReport {
    Vector x_star;
    double f_star = 0.0;
    double pg_norm = 0.0;
    SolveStatus status = SolveStatus::IterLimit;
    int iterations = 0;
    long cg_iterations = 0;
    long f_evals = 0;
    double wall_time = 0.0;
};

inline Vector clip(Vector x, const Vector& l, const Vector& u) {
    orc_clip(int(x.size()), x.data(), l.data(), u.data());
    return x;
}
inline double projected_gradient_norm(const Vector& x, const Vector& g, const Vector& l, const Vector& u) {
    return orc_pgnorm(int(x.size()), x.data(), g.data(), l.data(), u.data());
}
template <BoundedProblem P>
double projected_gradient_norm(const P& p, const Vector& x) {
    return projected_gradient_norm(x, p.eval_grad(x), p.lower(), p.upper());
}
inline Vector gpstep(const Vector& x, double alpha, const Vector& w, const Vector& l, const Vector& u) {
    Vector s(x.size());
    orc_gpstep(int(x.size()), x.data(), alpha, w.data(), l.data(), u.data(), s.data());
    return s;
}
struct BreakpointInfo {
    int count = 0;
    double min = 0.0;
    double max = 0.0;
};
inline BreakpointInfo breakpt(const Vector& x, const Vector& w, const Vector& l, const Vector& u) {
    BreakpointInfo b;
    orc_breakpt(int(x.size()), x.data(), w.data(), l.data(), u.data(), &b.count, &b.min, &b.max);
    return b;
}
inline double trqsol(const Vector& x, const Vector& w, double delta) {
    double s;
    if (orc_trqsol(int(x.size()), x.data(), w.data(), delta, &s))
        throw std::invalid_argument("trqsol: direction is zero, no intersection");
    return s;
}
struct CauchyStep {
    double alpha = 1.0;
    Vector s;
};
inline CauchyStep cauchy(const Vector& x, const Vector& g, const DenseMatrix& A, const Vector& l,
                         const Vector& u, double delta, const TronConfig& cfg, double alpha_start = 1.0) {
    const tb_tron_config c = cfg.c();
    CauchyStep cs{1.0, Vector(x.size())};
    if (orc_cauchy(int(x.size()), x.data(), g.data(), A.data(), l.data(), u.data(), delta, &c,
                   alpha_start, &cs.alpha, cs.s.data()))
        throw EvaluationError("cauchy: non-finite quadratic model value");
    return cs;
}
template <BoundedProblem P>
CauchyStep cauchy(const P& p, const Vector& x, const Vector& g, const DenseMatrix& A, double delta,
                  const TronConfig& cfg = {}) {
    return cauchy(x, g, A, p.lower(), p.upper(), delta, cfg);
}
inline std::vector<int> select_free_set(const Vector& x, const Vector& l, const Vector& u) {
    std::vector<int> f(x.size());
    f.resize(orc_select_free_set(int(x.size()), x.data(), l.data(), u.data(), f.data()));
    return f;
}
enum class CgStatus { Converged, Boundary, NegCurve, IterCap };
struct CgResult {
    Vector step;
    CgStatus status = CgStatus::IterCap;
    int iterations = 0;
    double rel_residual = 0.0;
};
inline CgResult precond_cg(const DenseMatrix& A, const Vector& g_free, const DenseMatrix& L, double delta,
                           const TronConfig& cfg = {}) {
    const int n = A.dim();
    if (int(g_free.size()) != n) throw std::invalid_argument("precond_cg: dimension mismatch");
    const tb_tron_config c = cfg.c();
    CgResult r;
    r.step.resize(n);
    int st = 0;
    const int rc = orc_precond_cg(n, A.data(), g_free.data(), L.data(), delta, &c, r.step.data(), &st,
                                  &r.iterations, &r.rel_residual);
    if (rc == TB_STATUS_ZERO_DIRECTION) throw std::invalid_argument("trqsol: direction is zero");
    if (rc == TB_STATUS_SINGULAR_FACTOR) throw SingularFactorError("trtrs: zero diagonal");
    r.status = static_cast<CgStatus>(st);
    return r;
}
struct LineSearchResult {
    double beta = 1.0;
    Vector x_next;
};
inline LineSearchResult projected_line_search(const Vector& x, const Vector& l, const Vector& u,
                                              const DenseMatrix& A, const Vector& g, const Vector& w,
                                              const TronConfig& cfg = {}) {
    const tb_tron_config c = cfg.c();
    LineSearchResult r{1.0, Vector(x.size())};
    orc_line_search(int(x.size()), x.data(), l.data(), u.data(), A.data(), g.data(), w.data(), &c,
                    &r.beta, r.x_next.data());
    return r;
}

namespace detail {
template <BoundedProblem P>
struct Tramp {
    static double f(void* c, const double* x) {
        const P& p = *static_cast<const P*>(c);
        return p.eval_f(Vector(x, x + p.dim()));
    }
    static void g(void* c, const double* x, double* out) {
        const P& p = *static_cast<const P*>(c);
        const Vector r = p.eval_grad(Vector(x, x + p.dim()));
        std::copy(r.begin(), r.end(), out);
    }
    static void h(void* c, const double* x, double* out) {
        const P& p = *static_cast<const P*>(c);
        const DenseMatrix r = p.eval_hess(Vector(x, x + p.dim()));
        std::copy(r.data(), r.data() + std::size_t(p.dim()) * p.dim(), out);
    }
};
}  // namespace detail

template <BoundedProblem P>
SolveReport solve(const P& p, Vector x0, const TronConfig& cfg = {}) {
    cfg.validate();
    const int n = p.dim();
    const Vector l = p.lower(), u = p.upper();
    if (int(x0.size()) != n || int(l.size()) != n || int(u.size()) != n)
        throw std::invalid_argument("solve: dimension mismatch");
    orc_problem op{n, l.data(), u.data(), &detail::Tramp<P>::f, &detail::Tramp<P>::g,
                   &detail::Tramp<P>::h, const_cast<void*>(static_cast<const void*>(&p))};
    const tb_tron_config c = cfg.c();
    SolveReport rep;
    rep.x_star.resize(n);
    orc_report r;
    const int rc = orc_solve(&op, x0.data(), &c, rep.x_star.data(), &r);
    if (rc == TB_STATUS_INVALID_BOUNDS) throw std::invalid_argument("solve: lower bound exceeds upper bound");
    if (rc == TB_STATUS_EVALUATION_ERROR) throw EvaluationError("cauchy: non-finite quadratic model value");
    if (rc == TB_STATUS_ZERO_DIRECTION) throw std::invalid_argument("trqsol: direction is zero");
    if (rc == TB_STATUS_SINGULAR_FACTOR) throw SingularFactorError("trtrs: zero diagonal");
    rep.f_star = r.f_star;
    rep.pg_norm = r.pg_norm;
    rep.status = static_cast<SolveStatus>(r.status);
    rep.iterations = r.iterations;
    rep.cg_iterations = r.cg_iterations;
    rep.f_evals = r.f_evals;
    return rep;
}
template <BoundedProblem P>
SolveReport solve(const P& p, const TronConfig& cfg = {}) {
    return solve(p, clip(Vector(p.dim(), 0.0), p.lower(), p.upper()), cfg);
}

}  // namespace tronbatch
