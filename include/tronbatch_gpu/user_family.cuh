// tronbatch_gpu/user_family.cuh — caller-defined problem families on the GPU,
// header-only: a caller's own __host__ __device__ f / grad / Hessian type
// instantiates the warp-per-problem TRON kernel in the caller's translation
// unit (compiled with nvcc -gencode arch=compute_100a,code=sm_100a
// --fmad=false), without rebuilding libtronbatch_b200.so.
//
// The reference accepts any BoundedProblem (tron.hpp:28-36: dim, lower,
// upper, eval_f, eval_grad, eval_hess) through solve_batch (batch.hpp:27-29).
// Host callables cannot run on the device, so a user family is a type with
// the three evaluations as __host__ __device__ static functions over
// (x, params, n):
//
//     struct MyFamily {
//         static constexpr int kMaxDim = 8;                                  // <= 32
//         __host__ __device__ static double f(const double* x, const double* p, int n);
//         __host__ __device__ static double grad(const double* x, const double* p, int n, int i);
//         __host__ __device__ static double hess(const double* x, const double* p, int n, int i, int j);
//     };
//
// UserProblem<MyFamily> satisfies the reference's BoundedProblem concept with
// the HOST side of the same functions, so one std::vector of them goes to the
// reference's tronbatch::solve_batch or to gpu::solve_batch_user below, and
// both run the same arithmetic (bitwise equal when the caller's functions
// are, e.g. compiled without FMA contraction on both sides).
//
// Device evaluation (tron_device.cuh tron_solve_one): every lane of the warp
// evaluates f (identical bits), lane i evaluates gradient component i and
// Hessian row i; evaluations happen only at the point of the latest f, as in
// the reference (tron.hpp:474-476, 506, 532, 489).  Dimensions up to 32 (the
// warp form); flop counting is not available for user families.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../paper_2106_14995_b200/csrc/tron_device.cuh"
#include "../tb_capi.h"

#if defined(__has_include)
#if __has_include("tronbatch/batch.hpp")
#include "tronbatch/batch.hpp"
#define TB_USER_FAMILY_HAVE_REFERENCE_TYPES 1
#endif
#endif

namespace tronbatch::gpu {

// the device side of a user family, in the solver's family interface
template <class UF, int D, bool COUNT>
struct UserFamily {
    using W_t = tbdev::Warp<D, COUNT>;
    __device__ __forceinline__ void bind(double*) {}
    __device__ __forceinline__ static long long flops(int, int) { return 0; }
    __device__ __forceinline__ void prepare(W_t& W, double x) {
        if (W.lane < W.n) W.xs[W.lane] = x;
        __syncwarp();
    }
    __device__ __forceinline__ double f(W_t& W) { return UF::f(W.xs, W.prm, W.n); }
    __device__ __forceinline__ double grad(W_t& W) {
        return W.lane < W.n ? UF::grad(W.xs, W.prm, W.n, W.lane) : 0.0;
    }
    __device__ __forceinline__ void hess(W_t& W) {
        if (W.lane < W.n)
            for (int j = 0; j < W.n; ++j) W.A[W.lane + j * D] = UF::hess(W.xs, W.prm, W.n, W.lane, j);
        __syncwarp();
    }
};

template <class UF, int D>
__global__ void __launch_bounds__(32, tbdev::WarpMinBlocks<D>::value)
    user_family_kernel(const __grid_constant__ tbdev::KernelArgs a) {
    extern __shared__ double smem[];
    const long long pid = blockIdx.x;
    if (pid >= a.count) return;
    tbdev::tron_solve_one<-1, D, false, UserFamily<UF, D, false>>(a, pid, smem);
}

template <class UF, int D>
cudaError_t launch_user_d(const tbdev::KernelArgs& a, cudaStream_t stream) {
    const size_t bytes = sizeof(double) * (size_t)(tbdev::SmemLayout<D>::fixed() + ((a.nparams + 1) & ~1));
    auto kern = user_family_kernel<UF, D>;
    if (bytes > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        if (e != cudaSuccess) return e;
    }
    kern<<<(unsigned)a.count, 32, bytes, stream>>>(a);
    return cudaGetLastError();
}

// Device-resident batch (all pointers device memory, problem-major like
// tb_problem_batch / tb_batch_result; any result pointer may be null except
// status), enqueued on `stream`.  Returns cudaSuccess or the launch error;
// per-problem statuses >= TB_STATUS_EVALUATION_ERROR mark problems the
// reference would have thrown on (see solve_batch_user).
template <class UF>
cudaError_t launch_user_batch(int n, int64_t count, const double* x0, const double* lower, const double* upper,
                              const double* params, int64_t params_stride, int nparams, const tb_tron_config& cfg,
                              double* x_star, double* f_star, double* pg_norm, int32_t* status, int32_t* iterations,
                              int64_t* cg_iterations, int64_t* f_evals, double* wall_time, cudaStream_t stream) {
    static_assert(UF::kMaxDim >= 1 && UF::kMaxDim <= 32, "user families: 1 <= kMaxDim <= 32 (warp form)");
    if (n < 1 || n > UF::kMaxDim || count < 0 || !status) return cudaErrorInvalidValue;
    if (count == 0) return cudaSuccess;
    tbdev::KernelArgs a{};
    a.n = n;
    a.nparams = nparams;
    a.count = count;
    a.stride = params_stride;
    a.x0 = x0;
    a.lo = lower;
    a.up = upper;
    a.prm = nparams > 0 ? params : nullptr;
    a.cfg = cfg;
    a.fast_forward = 1;
    a.extrap = 1.0 / cfg.interp_factor;
    a.x_star = x_star;
    a.f_star = f_star;
    a.pg_norm = pg_norm;
    a.status = status;
    a.iterations = iterations;
    a.cg_iterations = cg_iterations;
    a.f_evals = f_evals;
    a.wall_time = wall_time;
    a.route_count = count;
    // D = next of {4, 8, 16, 32} >= n (the library's warp-form instantiations)
    if (n <= 4) return launch_user_d<UF, 4>(a, stream);
    if constexpr (UF::kMaxDim > 4) {
        if (n <= 8) return launch_user_d<UF, 8>(a, stream);
    }
    if constexpr (UF::kMaxDim > 8) {
        if (n <= 16) return launch_user_d<UF, 16>(a, stream);
    }
    if constexpr (UF::kMaxDim > 16) return launch_user_d<UF, 32>(a, stream);
    return cudaErrorInvalidValue;
}

#ifdef TB_USER_FAMILY_HAVE_REFERENCE_TYPES
// A problem of family UF: the reference's BoundedProblem concept (tron.hpp:
// 28-36) over the HOST side of UF's functions, plus the parameters the device
// evaluates with.
template <class UF>
struct UserProblem {
    int n = 0;
    Vector l, u, prm;
    int dim() const { return n; }
    const Vector& lower() const { return l; }
    const Vector& upper() const { return u; }
    double eval_f(const Vector& x) const { return UF::f(x.data(), prm.data(), n); }
    Vector eval_grad(const Vector& x) const {
        Vector g(n);
        for (int i = 0; i < n; ++i) g[i] = UF::grad(x.data(), prm.data(), n, i);
        return g;
    }
    DenseMatrix eval_hess(const Vector& x) const {
        DenseMatrix a(n);
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) a(i, j) = UF::hess(x.data(), prm.data(), n, i, j);
        return a;
    }
};

// solve_batch (batch.hpp:27-29) for a user family on device 0: same
// arguments, result type and exceptions as the reference.
template <class UF>
BatchResult solve_batch_user(const std::vector<UserProblem<UF>>& problems, const std::vector<Vector>& x0s,
                             const TronConfig& cfg = {}) {
    if (problems.size() != x0s.size()) throw std::invalid_argument("solve_batch: problems and x0s length mismatch");
    cfg.validate();
    BatchResult out;
    const int64_t N = static_cast<int64_t>(problems.size());
    if (N == 0) return out;
    const int n = problems[0].dim();
    const int np = static_cast<int>(problems[0].prm.size());
    std::vector<double> h(N * (3 * n + std::max(np, 1)));
    double *hx = h.data(), *hl = hx + N * n, *hu = hl + N * n, *hp = hu + N * n;
    for (int64_t i = 0; i < N; ++i) {
        const auto& p = problems[i];
        if (p.dim() != n || static_cast<int>(x0s[i].size()) != n || static_cast<int>(p.prm.size()) != np)
            throw std::invalid_argument("solve: dimension mismatch");
        std::memcpy(hx + i * n, x0s[i].data(), sizeof(double) * n);
        std::memcpy(hl + i * n, p.l.data(), sizeof(double) * n);
        std::memcpy(hu + i * n, p.u.data(), sizeof(double) * n);
        if (np) std::memcpy(hp + i * np, p.prm.data(), sizeof(double) * np);
    }
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
    const size_t in_b = sizeof(double) * h.size();
    const size_t out_b = sizeof(double) * N * (n + 3) + sizeof(int32_t) * 2 * N + sizeof(int64_t) * 2 * N;
    char* d = nullptr;
    if (cudaMalloc(&d, in_b + out_b) != cudaSuccess) throw std::runtime_error("tronbatch::gpu: cudaMalloc failed");
    struct Free {
        char* p;
        ~Free() { cudaFree(p); }
    } guard{d};
    double* dx = reinterpret_cast<double*>(d);
    double *dl = dx + N * n, *du = dl + N * n, *dp = du + N * n;
    double* xs = reinterpret_cast<double*>(d + in_b);
    double *fs = xs + N * n, *pg = fs + N, *wt = pg + N;
    int64_t *cg = reinterpret_cast<int64_t*>(wt + N), *fe = cg + N;
    int32_t *st = reinterpret_cast<int32_t*>(fe + N), *it = st + N;
    cudaError_t e = cudaMemcpy(d, h.data(), in_b, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = launch_user_batch<UF>(n, N, dx, dl, du, dp, np, np, c, xs, fs, pg, st, it, cg, fe, wt, nullptr);
    std::vector<char> res(out_b);
    if (e == cudaSuccess) e = cudaMemcpy(res.data(), d + in_b, out_b, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) throw std::runtime_error(std::string("tronbatch::gpu: ") + cudaGetErrorString(e));
    const double* rx = reinterpret_cast<const double*>(res.data());
    const double *rf = rx + N * n, *rp = rf + N, *rw = rp + N;
    const int64_t *rc = reinterpret_cast<const int64_t*>(rw + N), *re = rc + N;
    const int32_t *rs = reinterpret_cast<const int32_t*>(re + N), *ri = rs + N;
    out.reports.resize(N);
    out.per_problem_time.assign(rw, rw + N);
    for (int64_t i = 0; i < N; ++i) {
        // batch.hpp:75-76: rethrow what the reference's solve would have thrown
        if (rs[i] == TB_STATUS_EVALUATION_ERROR) throw EvaluationError("cauchy: non-finite quadratic model value");
        if (rs[i] == TB_STATUS_SINGULAR_FACTOR) throw SingularFactorError("trtrs: zero diagonal");
        if (rs[i] == TB_STATUS_ZERO_DIRECTION) throw std::invalid_argument("trqsol: direction is zero");
        if (rs[i] == TB_STATUS_INVALID_BOUNDS) throw std::invalid_argument("solve: lower bound exceeds upper bound");
        SolveReport& s = out.reports[i];
        s.x_star.assign(rx + i * n, rx + (i + 1) * n);
        s.f_star = rf[i];
        s.pg_norm = rp[i];
        s.status = static_cast<SolveStatus>(rs[i]);
        s.iterations = ri[i];
        s.cg_iterations = rc[i];
        s.f_evals = re[i];
        s.wall_time = rw[i];
    }
    return out;
}
#endif

}  // namespace tronbatch::gpu
