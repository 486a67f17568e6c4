// admm.cu — device-resident component ADMM for AC-OPF,
// driving the batched TRON kernel for the branch subproblems.
//
// Per iteration, all on the device of this process:
//   admm_gen_kernel        generator closed form (all generators)
//   tron_solve_kernel      branch subproblems of this shard (warm start, in place);
//                          with line limits admm_auglag_fused_kernel runs each
//                          branch's augmented-Lagrangian loop in one launch
//   [exchange]             the caller all-gathers the branch solutions x
//                          (NCCL over NVLink when sharded; nothing when not)
//   admm_bus_warp_kernel   bus consensus + multipliers + residual terms (every
//                          bus, deterministic; residual max over this shard's
//                          buses -> the caller max-allreduces two doubles)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tb_capi.h"
#include "tb_admm.h"
#include "tb_admm_host.h"
#include "tron_device.cuh"
#include "tron_launch.h"
#include "tron_thread.cuh"

namespace {

// `stop` (may be null): set once tb_admm_run's iterations have converged; the
// stage kernels of later iterations return at once
__device__ __forceinline__ bool stopped(const int* stop) { return stop && *stop; }

__global__ void admm_gen_kernel(tb_admm_view v, const int* stop) {
    if (stopped(stop)) return;
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < v.n_gen) tb_admm_gen_update(&v, g);
}

// Generator and branch stages in ONE launch (they run
// concurrently): blocks [0, gen_blocks) update the generators, the others run
// one branch TRON solve per thread (tron_thread.cuh; in place: each thread
// reads its x0 before it writes x*).  The stages touch disjoint state.
constexpr int kThreadBlock = 64;
// The thread-form branch stage is ranked by start projected gradient
// (tron_order.cu) when the shard needs more than one wave of
// it (4 blocks of 64 threads per SM): the long branches then start in the
// first wave.  profiles/r02_ab_admm_order.txt: C5 (70,000 branches, ~1.9
// waves) 1.977 -> 1.877 ms per iteration; C4 (20,467, one wave) would lose
// 4 % (1.391 -> 1.445: every branch starts at once anyway), so it is not
// ranked.  0 disables.
#ifndef TB_ADMM_ORDER
#define TB_ADMM_ORDER 1
#endif
bool admm_ranked(long long cnt) { return TB_ADMM_ORDER && cnt > 4LL * kThreadBlock * tbdev::device_sm_count(); }
// The fused augmented-Lagrangian stage (dim 6, one warp per branch) is ranked
// like C2 beyond one wave of warps (profiles/r02_ab_admm_order.txt).
#ifndef TB_ADMM_AL_ORDER
#define TB_ADMM_AL_ORDER 1
#endif
bool admm_al_ranked(long long cnt) {
    return TB_ADMM_AL_ORDER && cnt > (long long)tbdev::WarpMinBlocks<6>::value * tbdev::device_sm_count();
}
#ifndef TB_ADMM_BRANCH_MINB
#define TB_ADMM_BRANCH_MINB 1  // resident 64-thread blocks per SM the register budget must allow
#endif
template <bool ORD>
__global__ void __launch_bounds__(kThreadBlock, TB_ADMM_BRANCH_MINB)
    admm_gen_branch_kernel(const __grid_constant__ tbdev::KernelArgs k, tb_admm_view v, int gen_blocks) {
    if (stopped(k.skip)) return;
    if ((int)blockIdx.x < gen_blocks) {
        const int g = blockIdx.x * kThreadBlock + threadIdx.x;
        if (g < v.n_gen) tb_admm_gen_update(&v, g);
        return;
    }
    const long long pid = (long long)(blockIdx.x - gen_blocks) * kThreadBlock + threadIdx.x;
    if (pid < k.count) tbdev::tron_solve_thread<4, TB_FAMILY_BRANCH>(k, ORD ? (long long)k.order[pid] : pid);
}

// first branch of [0, n) whose solve ended where the reference throws
// (status >= TB_STATUS_EVALUATION_ERROR), as a global branch index, into the
// sticky slot *first (atomicMin; ~0 = none)
__global__ void admm_status_scan_kernel(const int32_t* status, long long n, long long base,
                                        unsigned long long* first, const int* stop) {
    if (stopped(stop)) return;
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n && status[i] >= TB_STATUS_EVALUATION_ERROR) atomicMin(first, (unsigned long long)(base + i));
}

// tb_admm_update_consensus' export: residuals and the first failed branch of
// the shard (-1 none) as three doubles (the caller max-allreduces them across
// shards), and the failure record cleared for the next iteration
__global__ void admm_export_kernel(unsigned long long* res, double* out) {
    out[0] = __longlong_as_double((long long)res[0]);
    out[1] = __longlong_as_double((long long)res[1]);
    out[2] = res[2] == ~0ull ? -1.0 : (double)res[2];
    res[2] = ~0ull;
}

// tb_admm_run: after the bus pass of one iteration, append the residuals to
// the device history, stop once both tolerances hold (or a branch failed),
// and clear the residual slots for the next iteration
__global__ void admm_record_kernel(unsigned long long* res, double* hist, int* it, int cap, const double* tol,
                                   int* stop) {
    if (*stop) return;
    const double p = __longlong_as_double((long long)res[0]), d = __longlong_as_double((long long)res[1]);
    const int k = *it;
    if (k < cap) {
        hist[2 * k] = p;
        hist[2 * k + 1] = d;
    }
    *it = k + 1;
    if (res[2] != ~0ull) *stop = 2;
    else if (p <= tol[0] && d <= tol[1]) *stop = 1;
    res[0] = 0ull;
    res[1] = 0ull;
}

// residuals are non-negative doubles: unsigned max on the bit patterns
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* a, double x) {
    atomicMax(a, (unsigned long long)__double_as_longlong(x));
}

// The same bus pass (tb_admm_bus_update) with one warp per bus: lane k
// evaluates item k of the bus's canonical list (its generators, then its
// branch ends) -- the flows, quotients and per-coupling updates are
// independent per item -- and the ordered sums are formed from the staged
// terms in list order, so every sum, every multiplier and the residuals carry
// the bits of the serial form (max is order-free: NaN never enters, as in
// the serial `if (pr < d)`).  Serial per-bus work was the pass's latency
// (one thread walked a hub bus's ends with dependent loads and divisions).
constexpr int kBusWarps = 4;  // buses per block
__global__ void __launch_bounds__(32 * kBusWarps)
    admm_bus_warp_kernel(tb_admm_view v, int res_lo, int res_hi, unsigned long long* res, const int* stop) {
    if (stopped(stop)) return;
    __shared__ double stage[kBusWarps][8][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int b = blockIdx.x * kBusWarps + w;
    double (*T)[32] = stage[w];
    double pr = 0.0, du = 0.0;
    if (b < v.n_bus) {
        const int D = v.branch_dim;
        const int g0 = v.gen_ptr[b], ng = v.gen_ptr[b + 1] - g0;
        const int e0 = v.end_ptr[b], ne = v.end_ptr[b + 1] - e0;
        const int cnt = ng + ne;
        double SP = 0.0, WP = 0.0, SQ = 0.0, WQ = 0.0, Sw = 0.0, Rw = 0.0, St = 0.0, Rt = 0.0;
        // pass 1: terms per item (lane), ordered sums over the list
        for (int c0 = 0; c0 < cnt; c0 += 32) {
            const int k = c0 + lane;
            if (k < ng) {
                const int g = v.gen_idx[g0 + k];
                const double rp = v.gen_rp[g], rq = v.gen_rq[g];
                T[0][lane] = v.gen_p[g] + v.gen_lp[g] / rp;
                T[1][lane] = 1.0 / rp;
                T[2][lane] = v.gen_q[g] + v.gen_lq[g] / rq;
                T[3][lane] = 1.0 / rq;
            } else if (k < cnt) {
                const int e = v.end_idx[e0 + k - ng], l = e >> 1, end = e & 1;
                const double* prm = v.br_params + (long)l * TB_BR_NPARAMS;
                const double* x = v.br_x + (long)l * D;
                double base[8];
                tb_br_base(x, base);
                const int fp = 2 * end, fq = 2 * end + 1;
                T[0][lane] = tb_admm_flow(base, prm, fp) + prm[TB_BR_LAM + fp] / prm[TB_BR_RHO + fp];
                T[1][lane] = 1.0 / prm[TB_BR_RHO + fp];
                T[2][lane] = tb_admm_flow(base, prm, fq) + prm[TB_BR_LAM + fq] / prm[TB_BR_RHO + fq];
                T[3][lane] = 1.0 / prm[TB_BR_RHO + fq];
                const double vv = x[end];
                const double rw = prm[TB_BR_RHOW + end], rt = prm[TB_BR_RHOT + end];
                T[4][lane] = rw * (vv * vv + prm[TB_BR_LAMW + end] / rw);
                T[5][lane] = rw;
                T[6][lane] = rt * (x[2 + end] + prm[TB_BR_LAMT + end] / rt);
                T[7][lane] = rt;
            }
            __syncwarp();
            const int m = min(32, cnt - c0);
            for (int q = 0; q < m; ++q) {
                if (c0 + q < ng) {
                    SP += T[0][q];
                    WP += T[1][q];
                    SQ += T[2][q];
                    WQ += T[3][q];
                } else {
                    SP -= T[0][q];
                    WP += T[1][q];
                    SQ -= T[2][q];
                    WQ += T[3][q];
                    Sw += T[4][q];
                    Rw += T[5][q];
                    St += T[6][q];
                    Rt += T[7][q];
                }
            }
            __syncwarp();  // the next chunk rewrites the staging
        }
        // the bus's closed form (every lane, identical bits)
        const double pd = v.bus_pd[b], qd = v.bus_qd[b];
        const double aPw = -v.bus_gsh[b], aQw = v.bus_bsh[b];
        const double mbar = Sw / Rw;
        const double r1 = (SP + aPw * mbar) - pd;
        const double r2 = (SQ + aQw * mbar) - qd;
        const double A12 = (aPw * aQw) / Rw;
        double muP, muQ;
        if (A12 == 0.0) {
            muP = r1 / (WP + (aPw * aPw) / Rw);
            muQ = r2 / (WQ + (aQw * aQw) / Rw);
        } else {
            const double A11 = WP + (aPw * aPw) / Rw, A22 = WQ + (aQw * aQw) / Rw;
            const double det = A11 * A22 - A12 * A12;
            muP = (r1 * A22 - A12 * r2) / det;
            muQ = (A11 * r2 - A12 * r1) / det;
        }
        const double wt = mbar - (aPw * muP + aQw * muQ) / Rw;
        const double tt = St / Rt;
        // pass 2: consensus, multipliers and residual terms per item
        auto coupling = [&](double x, double xt_old, double xt_new, double rho, double& lam) {
            const double d_ = tb_admm_absd(rho * (xt_new - xt_old));
            if (du < d_) du = d_;
            const double g_ = x - xt_new;
            if (pr < tb_admm_absd(g_)) pr = tb_admm_absd(g_);
            lam += rho * g_;
        };
        for (int k = lane; k < cnt; k += 32) {
            if (k < ng) {
                const int g = v.gen_idx[g0 + k];
                const double rp = v.gen_rp[g], rq = v.gen_rq[g];
                const double ptn = (v.gen_p[g] + v.gen_lp[g] / rp) - muP / rp;
                const double qtn = (v.gen_q[g] + v.gen_lq[g] / rq) - muQ / rq;
                coupling(v.gen_p[g], v.gen_pt[g], ptn, rp, v.gen_lp[g]);
                coupling(v.gen_q[g], v.gen_qt[g], qtn, rq, v.gen_lq[g]);
                v.gen_pt[g] = ptn;
                v.gen_qt[g] = qtn;
            } else {
                const int e = v.end_idx[e0 + k - ng], l = e >> 1, end = e & 1;
                double* prm = v.br_params + (long)l * TB_BR_NPARAMS;
                const double* x = v.br_x + (long)l * D;
                double base[8];
                tb_br_base(x, base);
                const int fp = 2 * end, fq = 2 * end + 1;
                const double Fp = tb_admm_flow(base, prm, fp), Fq = tb_admm_flow(base, prm, fq);
                const double rP = prm[TB_BR_RHO + fp], rQ = prm[TB_BR_RHO + fq];
                const double Ftp = (Fp + prm[TB_BR_LAM + fp] / rP) + muP / rP;
                const double Ftq = (Fq + prm[TB_BR_LAM + fq] / rQ) + muQ / rQ;
                coupling(Fp, prm[TB_BR_TIL + fp], Ftp, rP, prm[TB_BR_LAM + fp]);
                coupling(Fq, prm[TB_BR_TIL + fq], Ftq, rQ, prm[TB_BR_LAM + fq]);
                prm[TB_BR_TIL + fp] = Ftp;
                prm[TB_BR_TIL + fq] = Ftq;
                const double vv = x[end];
                coupling(vv * vv, prm[TB_BR_WTIL + end], wt, prm[TB_BR_RHOW + end], prm[TB_BR_LAMW + end]);
                coupling(x[2 + end], prm[TB_BR_TTIL + end], tt, prm[TB_BR_RHOT + end], prm[TB_BR_LAMT + end]);
                prm[TB_BR_WTIL + end] = wt;
                prm[TB_BR_TTIL + end] = tt;
            }
        }
        if (lane == 0) {
            v.bus_wt[b] = wt;
            v.bus_tt[b] = tt;
        }
        if (b < res_lo || b >= res_hi) pr = du = 0.0;
    }
    const double p = tbdev::warp_max_nonneg(pr);
    const double d = tbdev::warp_max_nonneg(du);
    if (lane == 0) {
        atomic_max_nonneg(res + 0, p);
        atomic_max_nonneg(res + 1, d);
    }
}

__global__ void admm_cost_kernel(tb_admm_view v, double* out) {
    // deterministic order: one thread sums all generators ascending
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        double s = 0.0;
        for (int g = 0; g < v.n_gen; ++g) s += tb_admm_gen_cost(&v, g);
        *out = s;
    }
}

// ---- line limits: the augmented-Lagrangian loop of every branch, fused.
// One warp per branch runs its own loop (PAPER.md:271 anticipates an AL kernel
// on top of TRON): solve the d = 6 subproblem with the current (mu, xi), apply
// tb_admm_auglag_update, repeat until the branch is feasible or the round cap.
// Each branch's sequence of solves and updates is exactly the one of the
// synchronous rounds of the oracle (oracle/admm_oracle.c orc_branch_stage),
// so results are bit-identical, but a branch never waits for the slowest
// branch of a round.  x is solved in place (each solve reads x0 before it
// writes x*).  round_max receives the largest per-branch round count (= the
// number of synchronous rounds the oracle runs).
template <bool ORD>
__global__ void __launch_bounds__(32, tbdev::WarpMinBlocks<6>::value)
    admm_auglag_fused_kernel(const __grid_constant__ tbdev::KernelArgs a, double* prm_shard, double* eta_shard,
                             double xi0, double eta0, double feas_tol, double xi_max, int max_rounds,
                             int* round_max) {
    extern __shared__ double smem[];
    const long long k = blockIdx.x;
    if (k >= a.count || stopped(a.skip)) return;
    const long long pid = ORD ? (long long)a.order[k] : k;  // ORD: ranked launch (tron_order.cu)
    const int lane = threadIdx.x & 31;
    double* prm = prm_shard + pid * TB_BR_NPARAMS;
    if (lane == 0) {
        prm[TB_BR_XI] = xi0;
        eta_shard[pid] = eta0;
    }
    __syncwarp();
    int rounds = 0;
#pragma unroll 1
    for (int r = 0; r < max_rounds; ++r) {
        ++rounds;
        tbdev::tron_solve_one<TB_FAMILY_BRANCH, 6, false>(a, pid, smem);
        __syncwarp();
        int active = 0;
        if (lane == 0) active = tb_admm_auglag_update(a.x_star + pid * 6, prm, eta_shard + pid, feas_tol, xi_max);
        active = __shfl_sync(0xffffffffu, active, 0);
        __syncwarp();
        if (!active) break;
    }
    if (lane == 0) atomicMax(round_max, rounds);
}

__global__ void admm_round_accum_kernel(int* round_max, long long* total, const int* stop) {
    if (stopped(stop)) return;
    *total += *round_max;
    *round_max = 0;
}

__global__ void admm_line_viol_kernel(const double* x, const double* prm, int64_t n, unsigned long long* out) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double h[2];
    double v = l < n ? tb_admm_line_hmax(x + l * 6, prm + l * TB_BR_NPARAMS, h) : 0.0;
    if (!(v >= 0.0)) v = CUDART_INF;
    v = tbdev::warp_max_nonneg(v);
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(v));
}

thread_local std::string g_admm_err;

// selects `dev` for the scope of an entry point and restores the caller's device
struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        cudaSetDevice(dev);
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

int fail(int code, const std::string& m) {
    g_admm_err = m;
    return code;
}

}  // namespace

struct tb_admm {
    int device = 0;
    cudaStream_t stream = nullptr;
    tb_context* ctx = nullptr;
    tb_admm_view v{};           // device pointers
    std::vector<void*> allocs;  // owned device buffers
    double* x = nullptr;        // [n_rows][4] branch solutions (owned or caller's)
    double *lower = nullptr, *upper = nullptr;
    int32_t* status = nullptr;
    // res[0..1]: residual maxima (IEEE bits of non-negative doubles), res[2]:
    // first failed branch of the shard (sticky until the next step / run; ~0 none)
    unsigned long long* res = nullptr;
    double* cost = nullptr;
    // tb_admm_run: stop flag, iteration counter, residual history, tolerances,
    // and the captured CUDA graph of one iteration
    int* stop = nullptr;
    int* it_dev = nullptr;
    double* hist = nullptr;
    int hist_cap = 0;
    double* tol = nullptr;
    cudaGraphExec_t graph = nullptr;
    // stage timing of the latest iteration: [0] components start, [1] branch
    // stage done, [2] consensus done
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    int branch_form = TB_FORM_AUTO;
    int64_t br_lo = 0, br_hi = 0;
    int bus_lo = 0, bus_hi = 0;
    tb_tron_config tron{};
    long long iterations = 0;
    cudaStream_t last = nullptr;  // stream of the latest enqueued stage (tb_admm_get waits for it)
    // line limits (dim 6)
    int dim = 4;
    tb_admm_options opt{};
    double* eta = nullptr;
    int* round_max = nullptr;          // device: largest per-branch round count of this iteration
    long long* rounds_total = nullptr;  // device: sum over iterations
    void* ord = nullptr;                // launch-order workspace of the branch stage (tron_order.cu)
};

namespace {

template <typename T>
T* dalloc(tb_admm* a, size_t n, cudaError_t* err) {
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, sizeof(T) * (n ? n : 1));
    if (e != cudaSuccess) *err = e;
    else a->allocs.push_back(p);
    return static_cast<T*>(p);
}

template <typename T>
cudaError_t upload(T* dst, const T* src, size_t n) {
    return n ? cudaMemcpy(dst, src, sizeof(T) * n, cudaMemcpyHostToDevice) : cudaSuccess;
}

}  // namespace

extern "C" {

const char* tb_admm_last_error(void) { return g_admm_err.c_str(); }

void tb_admm_options_default(tb_admm_options* o) {
    std::memset(o, 0, sizeof(*o));
    o->rho_pq = 10.0;
    o->rho_va = 40.0;  // 4 * rho0
    o->shard_rank = 0;
    o->shard_count = 1;
    tb_config_default(&o->tron);
    o->line_limits = 0;
    o->auglag_max_iter = 20;
    o->auglag_xi0 = 10.0;
    o->auglag_xi_max = 1e8;
    o->auglag_eta0 = 0.1;
    o->auglag_feas_tol = 1e-6;
}

int tb_admm_create(const tb_admm_grid* gr, const tb_admm_options* opt, int32_t device, double* x_external,
                   tb_admm** out) {
    if (!gr || !opt || !out) return fail(TB_E_INVALID_ARGUMENT, "tb_admm_create: null argument");
    *out = nullptr;
    if (gr->n_bus < 1 || gr->n_branch < 1 || gr->n_gen < 0)
        return fail(TB_E_INVALID_ARGUMENT, "tb_admm_create: empty network");
    if (opt->shard_count < 1 || opt->shard_rank < 0 || opt->shard_rank >= opt->shard_count)
        return fail(TB_E_INVALID_ARGUMENT, "tb_admm_create: bad shard");
    if (!(opt->rho_pq > 0.0) || !(opt->rho_va > 0.0)) return fail(TB_E_INVALID_ARGUMENT, "tb_admm_create: rho must be > 0");
    if (tb_config_validate(&opt->tron) != TB_OK) return fail(TB_E_INVALID_ARGUMENT, tb_last_error());
    if (opt->line_limits &&
        (opt->auglag_max_iter < 1 || !(opt->auglag_xi0 > 0.0) || !(opt->auglag_xi_max >= opt->auglag_xi0) ||
         !(opt->auglag_eta0 > 0.0) || !(opt->auglag_feas_tol > 0.0)))
        return fail(TB_E_INVALID_ARGUMENT, "tb_admm_create: bad augmented-Lagrangian options");
    const int nb = gr->n_bus, ng = gr->n_gen, nl = gr->n_branch;
    for (int l = 0; l < nl; ++l)
        if (gr->br_from[l] < 0 || gr->br_from[l] >= nb || gr->br_to[l] < 0 || gr->br_to[l] >= nb)
            return fail(TB_E_INVALID_ARGUMENT, "tb_admm_create: branch endpoint out of range");
    for (int g = 0; g < ng; ++g)
        if (gr->gen_bus[g] < 0 || gr->gen_bus[g] >= nb)
            return fail(TB_E_INVALID_ARGUMENT, "tb_admm_create: generator bus out of range");

    // host-side initial state (shared init rules, tb_admm_host.h semantics)
    tb_admm_host_state hs;
    if (tb_admm_host_init(gr, opt, &hs) != 0) return fail(TB_E_INVALID_ARGUMENT, hs.err);
    for (int b = 0; b < nb; ++b)
        if (hs.end_ptr[b + 1] == hs.end_ptr[b]) {
            tb_admm_host_free(&hs);
            return fail(TB_E_INVALID_ARGUMENT, "tb_admm_create: bus " + std::to_string(b) + " has no branch");
        }

    if (opt->branch_form != TB_FORM_AUTO && opt->branch_form != TB_FORM_WARP) {
        tb_admm_host_free(&hs);
        return fail(TB_E_INVALID_ARGUMENT, "tb_admm_create: branch_form must be TB_FORM_AUTO or TB_FORM_WARP");
    }
    tb_admm* a = new tb_admm;
    a->device = device;
    a->tron = opt->tron;
    a->opt = *opt;
    a->branch_form = opt->branch_form;
    const int D = hs.dim;
    a->dim = D;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaError_t err = cudaSetDevice(device);
    if (err == cudaSuccess) err = cudaStreamCreateWithFlags(&a->stream, cudaStreamNonBlocking);
    const int64_t chunk = (nl + opt->shard_count - 1) / opt->shard_count;  // padded chunks for all-gather
    const int64_t rows = chunk * opt->shard_count;
    a->br_lo = std::min<int64_t>(nl, chunk * opt->shard_rank);
    a->br_hi = std::min<int64_t>(nl, chunk * (opt->shard_rank + 1));
    {
        const int base = nb / opt->shard_count, rem = nb % opt->shard_count;
        int lo = 0;
        for (int k = 0; k < opt->shard_rank; ++k) lo += base + (k < rem ? 1 : 0);
        a->bus_lo = lo;
        a->bus_hi = lo + base + (opt->shard_rank < rem ? 1 : 0);
    }
    tb_admm_view& v = a->v;
    v.n_bus = nb;
    v.n_gen = ng;
    v.n_branch = nl;
    v.branch_dim = D;
#define ALLOC_UP(field, T, n, src)                                       \
    do {                                                                 \
        T* p_ = dalloc<T>(a, (n), &err);                                 \
        if (err == cudaSuccess) err = upload<T>(p_, (src), (n));         \
        v.field = p_;                                                    \
    } while (0)
    if (err == cudaSuccess) {
        ALLOC_UP(bus_pd, double, nb, gr->bus_pd);
        ALLOC_UP(bus_qd, double, nb, gr->bus_qd);
        ALLOC_UP(bus_gsh, double, nb, gr->bus_gsh);
        ALLOC_UP(bus_bsh, double, nb, gr->bus_bsh);
        ALLOC_UP(bus_wt, double, nb, hs.bus_wt);
        ALLOC_UP(bus_tt, double, nb, hs.bus_tt);
        ALLOC_UP(gen_bus, int32_t, ng, gr->gen_bus);
        ALLOC_UP(gen_c2, double, ng, gr->gen_c2);
        ALLOC_UP(gen_c1, double, ng, gr->gen_c1);
        ALLOC_UP(gen_pmin, double, ng, gr->gen_pmin);
        ALLOC_UP(gen_pmax, double, ng, gr->gen_pmax);
        ALLOC_UP(gen_qmin, double, ng, gr->gen_qmin);
        ALLOC_UP(gen_qmax, double, ng, gr->gen_qmax);
        ALLOC_UP(gen_p, double, ng, hs.gen_p);
        ALLOC_UP(gen_q, double, ng, hs.gen_q);
        ALLOC_UP(gen_lp, double, ng, hs.gen_lp);
        ALLOC_UP(gen_lq, double, ng, hs.gen_lq);
        ALLOC_UP(gen_rp, double, ng, hs.gen_rp);
        ALLOC_UP(gen_rq, double, ng, hs.gen_rq);
        ALLOC_UP(gen_pt, double, ng, hs.gen_pt);
        ALLOC_UP(gen_qt, double, ng, hs.gen_qt);
        ALLOC_UP(br_from, int32_t, nl, gr->br_from);
        ALLOC_UP(br_to, int32_t, nl, gr->br_to);
        ALLOC_UP(br_params, double, (size_t)nl * TB_BR_NPARAMS, hs.br_params);
        ALLOC_UP(gen_ptr, int32_t, nb + 1, hs.gen_ptr);
        ALLOC_UP(gen_idx, int32_t, ng, hs.gen_idx);
        ALLOC_UP(end_ptr, int32_t, nb + 1, hs.end_ptr);
        ALLOC_UP(end_idx, int32_t, 2 * nl, hs.end_idx);
    }
#undef ALLOC_UP
    if (err == cudaSuccess) {
        if (x_external) a->x = x_external;
        else a->x = dalloc<double>(a, (size_t)rows * D, &err);
    }
    if (err == cudaSuccess) err = upload<double>(a->x, hs.br_x, (size_t)nl * D);
    if (err == cudaSuccess) {
        a->lower = dalloc<double>(a, (size_t)nl * D, &err);
        if (err == cudaSuccess) err = upload<double>(a->lower, hs.br_lower, (size_t)nl * D);
        a->upper = dalloc<double>(a, (size_t)nl * D, &err);
        if (err == cudaSuccess) err = upload<double>(a->upper, hs.br_upper, (size_t)nl * D);
        a->status = dalloc<int32_t>(a, (size_t)nl, &err);
        if ((D == 4 && admm_ranked(nl)) || (D == 6 && admm_al_ranked(nl)))
            a->ord = dalloc<char>(a, tbdev::order_ws_bytes(nl), &err);
        a->res = dalloc<unsigned long long>(a, 3, &err);
        a->cost = dalloc<double>(a, 1, &err);
        a->stop = dalloc<int>(a, 2, &err);
        if (err == cudaSuccess) a->it_dev = a->stop + 1;
        a->tol = dalloc<double>(a, 2, &err);
        if (err == cudaSuccess) err = cudaMemset(a->res, 0, 2 * sizeof(unsigned long long));
        if (err == cudaSuccess) err = cudaMemset(a->res + 2, 0xff, sizeof(unsigned long long));
        if (err == cudaSuccess) err = cudaMemset(a->stop, 0, 2 * sizeof(int));
        if (err == cudaSuccess) err = cudaMemset(a->status, 0, sizeof(int32_t) * (size_t)nl);
        for (int k = 0; k < 3 && err == cudaSuccess; ++k) err = cudaEventCreate(&a->ev[k]);
    }
    if (err == cudaSuccess && D == 6) {  // AL state
        a->eta = dalloc<double>(a, (size_t)nl, &err);
        a->round_max = dalloc<int>(a, 1, &err);
        a->rounds_total = dalloc<long long>(a, 1, &err);
        if (err == cudaSuccess) err = cudaMemset(a->round_max, 0, sizeof(int));
        if (err == cudaSuccess) err = cudaMemset(a->rounds_total, 0, sizeof(long long));
    }
    v.br_x = a->x;
    tb_admm_host_free(&hs);
    if (err == cudaSuccess) {
        const int32_t dev = device;
        if (tb_context_create(&dev, 1, &a->ctx) != TB_OK) err = cudaErrorUnknown;
    }
    cudaSetDevice(prev);
    if (err != cudaSuccess) {
        std::string m = std::string("tb_admm_create: ") + cudaGetErrorString(err);
        tb_admm_destroy(a);
        return fail(TB_E_CUDA, m);
    }
    *out = a;
    return TB_OK;
}

int tb_admm_destroy(tb_admm* a) {
    if (!a) return TB_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(a->device);
    if (a->stream) cudaStreamSynchronize(a->stream);
    if (a->graph) cudaGraphExecDestroy(a->graph);
    for (auto& e : a->ev)
        if (e) cudaEventDestroy(e);
    for (void* p : a->allocs) cudaFree(p);
    if (a->stream) cudaStreamDestroy(a->stream);
    if (a->ctx) tb_context_destroy(a->ctx);
    cudaSetDevice(prev);
    delete a;
    return TB_OK;
}

namespace {

bool capturing(cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}

// generator + branch stage of this shard on `st` (`stop`: tb_admm_run's flag
// or null), then the status scan into res[2]
int enqueue_components(tb_admm* a, cudaStream_t st, const int* stop) {
    const bool timed = !capturing(st);
    if (timed) cudaEventRecord(a->ev[0], st);
    const int64_t cnt = a->br_hi - a->br_lo;
    const int gen_blocks = (a->v.n_gen + kThreadBlock - 1) / kThreadBlock;
    tbdev::KernelArgs k{};
    k.nparams = TB_BR_NPARAMS;
    k.count = cnt;
    k.stride = TB_BR_NPARAMS;
    k.cfg = a->tron;
    k.fast_forward = 1;
    k.extrap = 1.0 / a->tron.interp_factor;
    k.prm = a->v.br_params + a->br_lo * TB_BR_NPARAMS;
    k.status = a->status + a->br_lo;
    k.skip = stop;
    k.form = a->branch_form;
    if (cnt > 0 && a->dim == 6) {
        // the whole augmented-Lagrangian loop of every branch in one launch
        if (a->v.n_gen > 0) {
            admm_gen_kernel<<<(a->v.n_gen + 127) / 128, 128, 0, st>>>(a->v, stop);
            tbdev::note_launches(1);
        }
        k.n = 6;
        k.x0 = a->x + a->br_lo * 6;
        k.lo = a->lower + a->br_lo * 6;
        k.up = a->upper + a->br_lo * 6;
        k.x_star = a->x + a->br_lo * 6;  // in place
        // (a thread-per-branch form of this loop measured 184 vs 283 iter/s on C4: the AL
        // rounds make the stage throughput-bound, where the warp form wins)
        const size_t smem = sizeof(double) * (size_t)(tbdev::SmemLayout<6>::fixed() + TB_BR_NPARAMS);
        if (a->ord && admm_al_ranked(cnt)) {
            const cudaError_t e = tbdev::launch_order(TB_FAMILY_BRANCH, k, a->ord, st, &k.order);
            if (e != cudaSuccess) return fail(TB_E_CUDA, cudaGetErrorString(e));
        }
        auto al = k.order ? admm_auglag_fused_kernel<true> : admm_auglag_fused_kernel<false>;
        al<<<(unsigned)cnt, 32, smem, st>>>(
            k, a->v.br_params + a->br_lo * TB_BR_NPARAMS, a->eta + a->br_lo, a->opt.auglag_xi0, a->opt.auglag_eta0,
            a->opt.auglag_feas_tol, a->opt.auglag_xi_max, a->opt.auglag_max_iter, a->round_max);
        admm_round_accum_kernel<<<1, 1, 0, st>>>(a->round_max, a->rounds_total, stop);
        tbdev::note_launches(2);
    } else if (a->branch_form == TB_FORM_AUTO) {
        // generators and one thread per branch (tron_thread.cuh) in one
        // launch: the stage waits for its slowest branch, whose latency this
        // form cuts
        k.n = 4;
        k.x0 = a->x + a->br_lo * 4;
        k.lo = a->lower + a->br_lo * 4;
        k.up = a->upper + a->br_lo * 4;
        k.x_star = a->x + a->br_lo * 4;  // in place: each thread reads its x0 first
        const long long blocks = gen_blocks + (cnt + kThreadBlock - 1) / kThreadBlock;
        if (a->ord && admm_ranked(cnt)) {
            const cudaError_t e = tbdev::launch_order(TB_FAMILY_BRANCH, k, a->ord, st, &k.order);
            if (e != cudaSuccess) return fail(TB_E_CUDA, cudaGetErrorString(e));
        }
        if (blocks > 0) {
            if (k.order) admm_gen_branch_kernel<true><<<(unsigned)blocks, kThreadBlock, 0, st>>>(k, a->v, gen_blocks);
            else admm_gen_branch_kernel<false><<<(unsigned)blocks, kThreadBlock, 0, st>>>(k, a->v, gen_blocks);
            tbdev::note_launches(1);
        }
    } else {
        // warp per branch (KernelForm.WARP) through the library's launcher
        if (a->v.n_gen > 0) {
            admm_gen_kernel<<<(a->v.n_gen + 127) / 128, 128, 0, st>>>(a->v, stop);
            tbdev::note_launches(1);
        }
        if (cnt > 0) {
            k.n = 4;
            k.x0 = a->x + a->br_lo * 4;
            k.lo = a->lower + a->br_lo * 4;
            k.up = a->upper + a->br_lo * 4;
            k.x_star = a->x + a->br_lo * 4;  // in place: each warp reads its x0 before writing x*
            k.route_count = cnt;
            const cudaError_t e = tbdev::launch_tron(TB_FAMILY_BRANCH, k, st);
            if (e != cudaSuccess) return fail(TB_E_CUDA, cudaGetErrorString(e));
        }
    }
    if (cnt > 0) {
        admm_status_scan_kernel<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(a->status + a->br_lo, cnt, a->br_lo,
                                                                             a->res + 2, stop);
        tbdev::note_launches(1);
    }
    if (timed) cudaEventRecord(a->ev[1], st);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TB_OK : fail(TB_E_CUDA, cudaGetErrorString(e));
}

int enqueue_consensus(tb_admm* a, cudaStream_t st, const int* stop) {
    admm_bus_warp_kernel<<<(a->v.n_bus + kBusWarps - 1) / kBusWarps, 32 * kBusWarps, 0, st>>>(a->v, a->bus_lo,
                                                                                             a->bus_hi, a->res, stop);
    tbdev::note_launches(1);
    if (!capturing(st)) cudaEventRecord(a->ev[2], st);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TB_OK : fail(TB_E_CUDA, cudaGetErrorString(e));
}

std::string branch_error_message(tb_admm* a, unsigned long long idx) {
    int32_t st = 0;
    cudaMemcpy(&st, a->status + idx, sizeof st, cudaMemcpyDeviceToHost);
    const char* what = st == TB_STATUS_EVALUATION_ERROR ? "EvaluationError"
                       : st == TB_STATUS_ZERO_DIRECTION ? "invalid_argument (trqsol: zero direction)"
                       : st == TB_STATUS_SINGULAR_FACTOR ? "SingularFactorError"
                                                         : "invalid_argument (bounds)";
    return "ADMM branch stage: branch " + std::to_string(idx) + " failed with status " + std::to_string(st) + " (" +
           what + ")";
}

}  // namespace

// generator update (all generators) + branch TRON on this shard, enqueued on
// `stream` (NULL: the ADMM's own stream); returns without synchronising.
// Branch failures are recorded on the device (tb_admm_branch_errors).
int tb_admm_solve_components(tb_admm* a, void* stream) {
    if (!a) return fail(TB_E_INVALID_ARGUMENT, "null admm");
    DeviceGuard guard(a->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : a->stream;
    a->last = st;
    return enqueue_components(a, st, nullptr);
}

// device branch-solution buffer [rows][4]; this shard owns rows [lo, hi);
// rows are padded to shard_count equal chunks of `chunk` rows for all-gather
int tb_admm_branch_solution(tb_admm* a, double** x_dev, int64_t* lo, int64_t* hi) {
    if (!a) return fail(TB_E_INVALID_ARGUMENT, "null admm");
    *x_dev = a->x;
    *lo = a->br_lo;
    *hi = a->br_hi;
    return TB_OK;
}

// bus consensus + multipliers over every bus (needs the complete x); if
// res3_dev is non-NULL: residual maxima over this shard's buses in
// res3_dev[0..1] and the shard's first failed branch (-1 none) in res3_dev[2]
// (device doubles); enqueued on `stream`.
int tb_admm_update_consensus(tb_admm* a, void* stream, double* res3_dev) {
    if (!a) return fail(TB_E_INVALID_ARGUMENT, "null admm");
    DeviceGuard guard(a->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : a->stream;
    a->last = st;
    cudaMemsetAsync(a->res, 0, 2 * sizeof(unsigned long long), st);
    int rc = enqueue_consensus(a, st, nullptr);
    if (rc) return rc;
    if (res3_dev) {
        admm_export_kernel<<<1, 1, 0, st>>>(a->res, res3_dev);
        tbdev::note_launches(1);
    }
    ++a->iterations;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TB_OK : fail(TB_E_CUDA, cudaGetErrorString(e));
}

// first failed branch of this shard since the last call (blocking; -1: none),
// and its status; clears the record
int tb_admm_branch_errors(tb_admm* a, int64_t* first_bad, int32_t* status) {
    if (!a || !first_bad) return fail(TB_E_INVALID_ARGUMENT, "null argument");
    DeviceGuard guard(a->device);
    if (a->last && a->last != a->stream) cudaStreamSynchronize(a->last);
    unsigned long long idx = ~0ull;
    cudaError_t e = cudaMemcpy(&idx, a->res + 2, sizeof idx, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemset(a->res + 2, 0xff, sizeof idx);
    if (e != cudaSuccess) return fail(TB_E_CUDA, cudaGetErrorString(e));
    *first_bad = idx == ~0ull ? -1 : (int64_t)idx;
    if (status) {
        *status = 0;
        if (idx != ~0ull) cudaMemcpy(status, a->status + idx, sizeof *status, cudaMemcpyDeviceToHost);
    }
    return TB_OK;
}

// one full iteration in a single process (no exchange needed), blocking;
// primal / dual residuals to host.  TB_E_PROBLEM if a branch solve ended
// where the reference would throw (the state is advanced regardless).
int tb_admm_step(tb_admm* a, double* primal, double* dual) {
    if (!a) return fail(TB_E_INVALID_ARGUMENT, "null admm");
    DeviceGuard guard(a->device);
    a->last = a->stream;
    cudaMemsetAsync(a->res + 2, 0xff, sizeof(unsigned long long), a->stream);
    int rc = enqueue_components(a, a->stream, nullptr);
    if (rc) return rc;
    rc = tb_admm_update_consensus(a, nullptr, nullptr);
    if (rc) return rc;
    unsigned long long r[3];
    cudaError_t e = cudaMemcpyAsync(r, a->res, sizeof r, cudaMemcpyDeviceToHost, a->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(a->stream);
    if (e != cudaSuccess) return fail(TB_E_CUDA, cudaGetErrorString(e));
    if (primal) std::memcpy(primal, &r[0], sizeof(double));
    if (dual) std::memcpy(dual, &r[1], sizeof(double));
    if (r[2] != ~0ull) return fail(TB_E_PROBLEM, branch_error_message(a, r[2]));
    return TB_OK;
}

// admm_solve on one process without a host round trip per
// iteration: one iteration (stages + residual record) is captured once as a
// CUDA graph and replayed; the record kernel raises a device stop flag at the
// first iteration whose residuals are both <= tol (or whose branch stage
// failed), and every stage kernel of the iterations enqueued after it returns
// at once, so the state equals stopping exactly there.  The host checks the
// flag every `check_every` iterations.  hist_out: [max_iter][2] residuals
// (may be NULL); *iters_out: iterations run.
int tb_admm_run(tb_admm* a, int32_t max_iter, double tol_primal, double tol_dual, int32_t check_every,
                double* hist_out, int32_t* iters_out) {
    if (!a || !iters_out) return fail(TB_E_INVALID_ARGUMENT, "null argument");
    if (max_iter < 0 || check_every < 1) return fail(TB_E_INVALID_ARGUMENT, "tb_admm_run: bad max_iter / check_every");
    if (a->br_lo != 0 || a->br_hi != a->v.n_branch)
        return fail(TB_E_INVALID_ARGUMENT, "tb_admm_run: single-shard ADMM only (sharded runs exchange per iteration)");
    DeviceGuard guard(a->device);
    cudaStream_t st = a->stream;
    a->last = st;
    cudaError_t e = cudaSuccess;
    if (max_iter > a->hist_cap) {
        if (a->graph) {  // the graph holds the old history pointer
            cudaGraphExecDestroy(a->graph);
            a->graph = nullptr;
        }
        if (a->hist) {  // release the smaller history (no launch uses it any more: the stream is idle)
            cudaStreamSynchronize(st);
            a->allocs.erase(std::remove(a->allocs.begin(), a->allocs.end(), static_cast<void*>(a->hist)),
                            a->allocs.end());
            cudaFree(a->hist);
            a->hist = nullptr;
            a->hist_cap = 0;
        }
        // at least 64 iterations so short runs do not rebuild the graph each time
        const int cap = std::max(max_iter, 64);
        a->hist = dalloc<double>(a, (size_t)2 * cap, &e);
        if (e != cudaSuccess) return fail(TB_E_CUDA, cudaGetErrorString(e));
        a->hist_cap = cap;
    }
    const double tol[2] = {tol_primal, tol_dual};
    e = cudaMemcpyAsync(a->tol, tol, sizeof tol, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(a->stop, 0, 2 * sizeof(int), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(a->res, 0, 2 * sizeof(unsigned long long), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(a->res + 2, 0xff, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return fail(TB_E_CUDA, cudaGetErrorString(e));
    if (!a->graph) {
        cudaGraph_t g = nullptr;
        e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) return fail(TB_E_CUDA, cudaGetErrorString(e));
        int rc = enqueue_components(a, st, a->stop);
        if (rc == TB_OK) rc = enqueue_consensus(a, st, a->stop);
        if (rc == TB_OK) {
            admm_record_kernel<<<1, 1, 0, st>>>(a->res, a->hist, a->it_dev, a->hist_cap, a->tol, a->stop);
            tbdev::note_launches(1);
        }
        e = cudaStreamEndCapture(st, &g);
        if (rc) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        if (e == cudaSuccess) e = cudaGraphInstantiate(&a->graph, g, 0);
        if (g) cudaGraphDestroy(g);
        if (e != cudaSuccess) return fail(TB_E_CUDA, cudaGetErrorString(e));
    }
    int done = 0, it = 0, stop = 0;
    while (done < max_iter) {
        const int k = std::min<int>(check_every, max_iter - done);
        for (int i = 0; i < k && e == cudaSuccess; ++i) e = cudaGraphLaunch(a->graph, st);
        done += k;
        int flags[2] = {0, 0};
        if (e == cudaSuccess) e = cudaMemcpyAsync(flags, a->stop, sizeof flags, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return fail(TB_E_CUDA, cudaGetErrorString(e));
        stop = flags[0];
        it = flags[1];
        if (stop) break;
    }
    a->iterations += it;
    *iters_out = it;
    if (hist_out && it > 0) {
        e = cudaMemcpy(hist_out, a->hist, sizeof(double) * 2 * (size_t)it, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return fail(TB_E_CUDA, cudaGetErrorString(e));
    }
    if (stop == 2) {
        unsigned long long idx = ~0ull;
        cudaMemcpy(&idx, a->res + 2, sizeof idx, cudaMemcpyDeviceToHost);
        return fail(TB_E_PROBLEM, branch_error_message(a, idx));
    }
    return TB_OK;
}

// copy a state array to host: what = TB_ADMM_*
int tb_admm_get(tb_admm* a, int32_t what, void* host_out) {
    if (!a || !host_out) return fail(TB_E_INVALID_ARGUMENT, "null argument");
    DeviceGuard guard(a->device);
    if (a->last && a->last != a->stream) cudaStreamSynchronize(a->last);  // stages enqueued on a caller stream
    cudaStreamSynchronize(a->stream);
    const tb_admm_view& v = a->v;
    const void* src = nullptr;
    size_t bytes = 0;
    switch (what) {
        case TB_ADMM_GEN_P: src = v.gen_p; bytes = sizeof(double) * v.n_gen; break;
        case TB_ADMM_GEN_Q: src = v.gen_q; bytes = sizeof(double) * v.n_gen; break;
        case TB_ADMM_GEN_PT: src = v.gen_pt; bytes = sizeof(double) * v.n_gen; break;
        case TB_ADMM_GEN_QT: src = v.gen_qt; bytes = sizeof(double) * v.n_gen; break;
        case TB_ADMM_GEN_LP: src = v.gen_lp; bytes = sizeof(double) * v.n_gen; break;
        case TB_ADMM_GEN_LQ: src = v.gen_lq; bytes = sizeof(double) * v.n_gen; break;
        case TB_ADMM_BUS_WT: src = v.bus_wt; bytes = sizeof(double) * v.n_bus; break;
        case TB_ADMM_BUS_TT: src = v.bus_tt; bytes = sizeof(double) * v.n_bus; break;
        case TB_ADMM_BRANCH_X: src = a->x; bytes = sizeof(double) * a->dim * (size_t)v.n_branch; break;
        case TB_ADMM_AUGLAG_ROUNDS: {
            if (a->dim != 6) {
                const int64_t z = 0;
                std::memcpy(host_out, &z, sizeof z);
                return TB_OK;
            }
            src = a->rounds_total;
            bytes = sizeof(long long);
            break;
        }
        case TB_ADMM_LINE_VIOL: {
            if (a->dim != 6) return fail(TB_E_INVALID_ARGUMENT, "tb_admm_get: line limits are off");
            unsigned long long* m = reinterpret_cast<unsigned long long*>(a->cost);
            cudaMemsetAsync(m, 0, sizeof *m, a->stream);
            admm_line_viol_kernel<<<(unsigned)((v.n_branch + 127) / 128), 128, 0, a->stream>>>(a->x, v.br_params,
                                                                                               v.n_branch, m);
            src = a->cost;
            bytes = sizeof(double);
            break;
        }
        case TB_ADMM_BRANCH_PARAMS: src = v.br_params; bytes = sizeof(double) * TB_BR_NPARAMS * (size_t)v.n_branch; break;
        case TB_ADMM_BRANCH_STATUS: src = a->status; bytes = sizeof(int32_t) * (size_t)v.n_branch; break;
        case TB_ADMM_STAGE_TIMES: {  // seconds: [components (generators + branch TRON), consensus pass]
            float ms[2] = {0.f, 0.f};
            cudaError_t e = cudaEventSynchronize(a->ev[2]);
            if (e == cudaSuccess) e = cudaEventElapsedTime(&ms[0], a->ev[0], a->ev[1]);
            if (e == cudaSuccess) e = cudaEventElapsedTime(&ms[1], a->ev[1], a->ev[2]);
            if (e != cudaSuccess) return fail(TB_E_CUDA, cudaGetErrorString(e));
            const double t[2] = {1e-3 * ms[0], 1e-3 * ms[1]};
            std::memcpy(host_out, t, sizeof t);
            return TB_OK;
        }
        case TB_ADMM_COST: {
            admm_cost_kernel<<<1, 1, 0, a->stream>>>(a->v, a->cost);
            src = a->cost;
            bytes = sizeof(double);
            break;
        }
        default: return fail(TB_E_INVALID_ARGUMENT, "tb_admm_get: unknown field");
    }
    cudaError_t e = cudaStreamSynchronize(a->stream);  // the COST / LINE_VIOL kernels ran on a->stream
    if (e == cudaSuccess) e = cudaMemcpy(host_out, src, bytes, cudaMemcpyDeviceToHost);
    return e == cudaSuccess ? TB_OK : fail(TB_E_CUDA, cudaGetErrorString(e));
}

}  // extern "C"
