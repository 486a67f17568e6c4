// oracle/compat/tronbatch/batch.hpp — TEST INFRASTRUCTURE ONLY.
// The reference's batch.hpp API over the plain-C oracle; Hs45Problem
// evaluates the shared device twin (csrc/tb_families.h) so the reference's
// hs45 tests pin that twin too.
#pragma once
#include <string>
#include <vector>

#include "../../../paper_2106_14995_b200/csrc/tb_families.h"
#include "tronbatch/tron.hpp"

namespace tronbatch {

inline constexpr int kDefaultCapacity = 64;

struct BatchResult {
    std::vector<SolveReport> reports;
    std::vector<double> per_problem_time;
    std::vector<double> partition_times;
    double batch_wall_time = 0.0;
};

template <BoundedProblem P>
BatchResult solve_batch(const std::vector<P>& problems, const std::vector<Vector>& x0s,
                        const TronConfig& cfg = {}, int workers = 1) {
    if (workers < 1) throw std::invalid_argument("solve_batch: workers must be >= 1");
    if (problems.size() != x0s.size())
        throw std::invalid_argument("solve_batch: problems and x0s length mismatch");
    cfg.validate();
    BatchResult out;
    out.per_problem_time.assign(problems.size(), 0.0);
    out.partition_times.assign(workers, 0.0);
    for (std::size_t i = 0; i < problems.size(); ++i) out.reports.push_back(solve(problems[i], x0s[i], cfg));
    return out;
}

struct ImbalanceStats {
    std::vector<double> nu_per_iter;
    double nu_max = 0.0;
    double nu_min = 0.0;
    double nu_mean = 0.0;
};

inline ImbalanceStats imbalance(const std::vector<std::vector<double>>& t) {
    if (t.empty()) throw std::invalid_argument("imbalance: need at least one iteration");
    const int parts = int(t[0].size());
    std::vector<double> flat;
    for (const auto& row : t) {
        if (int(row.size()) != parts || parts < 2) throw std::invalid_argument("imbalance: need at least 2 partitions");
        flat.insert(flat.end(), row.begin(), row.end());
    }
    ImbalanceStats s;
    s.nu_per_iter.resize(t.size());
    if (orc_imbalance(flat.data(), int(t.size()), parts, s.nu_per_iter.data(), &s.nu_max, &s.nu_min, &s.nu_mean))
        throw std::invalid_argument("imbalance: partition times must be positive");
    return s;
}

class Hs45Problem {
public:
    explicit Hs45Problem(int n, int capacity = kDefaultCapacity) : n_(n) {
        if (n < 1 || n > capacity) throw std::invalid_argument("Hs45Problem: dimension out of capacity");
        l_.assign(n, 0.0);
        u_.resize(n);
        for (int i = 0; i < n; ++i) u_[i] = double(i + 1);
    }
    int dim() const { return n_; }
    const Vector& lower() const { return l_; }
    const Vector& upper() const { return u_; }
    Vector default_start() const { return scal(0.5, u_); }
    double eval_f(const Vector& x) const { return tb_hs45_f(x.data(), n_); }
    Vector eval_grad(const Vector& x) const {
        Vector g(n_);
        tb_family_grad(TB_FAMILY_HS45, x.data(), nullptr, n_, g.data());
        return g;
    }
    DenseMatrix eval_hess(const Vector& x) const {
        DenseMatrix h(n_);
        tb_family_hess(TB_FAMILY_HS45, x.data(), nullptr, n_, h.data());
        return h;
    }

private:
    int n_ = 0;
    Vector l_, u_;
};

inline Hs45Problem make_hs45(int n, int capacity = kDefaultCapacity) { return Hs45Problem(n, capacity); }

}  // namespace tronbatch
