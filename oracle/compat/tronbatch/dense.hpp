// oracle/compat/tronbatch/dense.hpp — TEST INFRASTRUCTURE ONLY.
// The reference's dense.hpp API (/root/reference/proj/include/tronbatch/
// dense.hpp) re-exposed over the plain-C oracle (oracle/tron_oracle.c), so the
// reference's own unit tests compile unmodified against the restatement
// (-I oracle/compat shadows the reference include dir).  Argument checks that
// the reference performs in C++ (dimension mismatches) are repeated here.
#pragma once
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../tron_oracle.h"

namespace tronbatch {

using Vector = std::vector<double>;

class FactorizationError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class SingularFactorError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

class DenseMatrix {
public:
    DenseMatrix() = default;
    explicit DenseMatrix(int n, double value = 0.0) : n_(n), data_(std::size_t(n) * n, value) {
        if (n < 1) throw std::invalid_argument("DenseMatrix: dimension must be >= 1");
    }
    static DenseMatrix identity(int n) {
        DenseMatrix a(n);
        for (int i = 0; i < n; ++i) a(i, i) = 1.0;
        return a;
    }
    int dim() const { return n_; }
    double& operator()(int i, int j) { return data_[std::size_t(i) + std::size_t(j) * n_]; }
    double operator()(int i, int j) const { return data_[std::size_t(i) + std::size_t(j) * n_]; }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    double max_abs() const { return orc_max_abs(n_, data_.data()); }

private:
    int n_ = 0;
    std::vector<double> data_;
};

namespace detail {
inline void require_same_size(const Vector& x, const Vector& y, const char* where) {
    if (x.size() != y.size()) throw std::invalid_argument(std::string(where) + ": dimension mismatch");
}
}  // namespace detail

inline Vector axpy(double alpha, const Vector& x, Vector y) {
    detail::require_same_size(x, y, "axpy");
    orc_axpy(int(y.size()), alpha, x.data(), y.data());
    return y;
}
inline double dot(const Vector& x, const Vector& y) {
    detail::require_same_size(x, y, "dot");
    return orc_dot(int(x.size()), x.data(), y.data());
}
inline double nrm2(const Vector& x) { return orc_nrm2(int(x.size()), x.data()); }
inline Vector scal(double alpha, Vector x) {
    orc_scal(int(x.size()), alpha, x.data());
    return x;
}
inline Vector copy(const Vector& x) { return x; }
inline Vector gemv(double alpha, const DenseMatrix& A, const Vector& x, double beta, Vector y,
                   bool transpose = false) {
    const int n = A.dim();
    if (int(x.size()) != n || int(y.size()) != n) throw std::invalid_argument("gemv: dimension mismatch");
    orc_gemv(n, alpha, A.data(), x.data(), beta, y.data(), transpose ? 1 : 0);
    return y;
}
inline DenseMatrix ccfs(DenseMatrix A, double alpha) {
    orc_ccfs(A.dim(), A.data(), alpha);
    return A;
}

struct CholeskyResult {
    DenseMatrix L;
    double shift;
};

inline CholeskyResult ccf(const DenseMatrix& A) {
    CholeskyResult r{DenseMatrix(A.dim()), 0.0};
    if (orc_ccf(A.dim(), A.data(), r.L.data(), &r.shift))
        throw FactorizationError("ccf: factorization failed");
    return r;
}
inline CholeskyResult ccf_right_looking(const DenseMatrix& A) {
    CholeskyResult r{DenseMatrix(A.dim()), 0.0};
    if (orc_ccf_right(A.dim(), A.data(), r.L.data(), &r.shift))
        throw FactorizationError("ccf: factorization failed");
    return r;
}
inline Vector trtrs(const DenseMatrix& L, Vector b, bool transpose = false) {
    const int n = L.dim();
    if (int(b.size()) != n) throw std::invalid_argument("trtrs: dimension mismatch");
    if (orc_trtrs(n, L.data(), b.data(), transpose ? 1 : 0))
        throw SingularFactorError("trtrs: zero diagonal");
    return b;
}

}  // namespace tronbatch
