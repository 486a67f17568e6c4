// capi.cu — the C ABI (include/tb_capi.h) over the device TRON kernels.
//
// solve_batch (batch.hpp:27-78) semantics: validate the config, split the
// batch into contiguous even partitions in input order (batch.hpp:61-70),
// one partition per device, solve each on its own stream, and surface the
// first (in input order) problem that the reference would have thrown on.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif

#include "../../include/tb_capi.h"
#include "tb_families.h"
#include "tron_device.cuh"
#include "tron_launch.h"

namespace {

thread_local std::string g_err;

int set_err(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CUDA_TRY(expr)                                                                     \
    do {                                                                                   \
        cudaError_t e_ = (expr);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return set_err(TB_E_CUDA, "%s failed: %s", #expr, cudaGetErrorString(e_));     \
    } while (0)

// device buffer that only grows
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) {
            // work queued on any stream of this device may still use the old
            // buffer (async solves): drain the device before releasing it
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) return e;
            cudaFree(p);
        }
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

// page-locked host buffer that only grows (library-owned staging for pageable
// caller buffers)
struct HostBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFreeHost(p);  // tb_solve_batch is blocking: no copy is pending
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocPortable);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
};

struct DevState {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t aux[8] = {};  // one stream per chunk of the host-buffer pipeline
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t fork = nullptr, join = nullptr;
    DevBuf in;   // x0, lower, upper, params
    DevBuf out;  // results
    DevBuf flag;
    DevBuf ws;   // block-kernel workspace (d > 16)
    HostBuf hin;   // pinned staging of pageable inputs (the device `in` layout)
    HostBuf hout;  // pinned staging of pageable outputs (the device `out` layout)
    // the last launch that used `ws` (block kernel): a later launch on any
    // stream waits for it, so overlapping async solves never share the
    // workspace's work counter and Hessian slices
    cudaEvent_t ws_ev = nullptr;
    DevBuf ord;                     // launch-order workspace (tron_order.cu)
    cudaEvent_t ord_ev = nullptr;   // its last user, like ws_ev
};

__global__ void first_error_kernel(const int32_t* status, long long count, unsigned long long* out) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < count && status[i] >= TB_STATUS_EVALUATION_ERROR) atomicMin(out, (unsigned long long)i);
}

}  // namespace

// Host threads of a context for its staging copies, started once (starting
// threads for every copy set costs ~0.1 ms, as much as the copies they share).
class HostPool {
public:
    explicit HostPool(int n) : nt_(n < 1 ? 1 : n) {
        for (int k = 1; k < nt_; ++k) th_.emplace_back([this, k] { loop(k); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    int size() const { return nt_; }
    // fn(k) for k in [0, t), t <= size(); the caller runs k = 0
    void run(int t, const std::function<void(int)>& fn) {
        if (t <= 1) {
            fn(0);
            return;
        }
        {
            std::lock_guard<std::mutex> g(m_);
            job_ = &fn;
            jobs_ = t;
            pending_ = nt_ - 1;
            ++gen_;
        }
        cv_.notify_all();
        fn(0);
        std::unique_lock<std::mutex> l(m_);
        done_.wait(l, [&] { return pending_ == 0; });
        job_ = nullptr;
    }

private:
    void loop(int k) {
        unsigned long long seen = 0;
        for (;;) {
            const std::function<void(int)>* job;
            int jobs;
            {
                std::unique_lock<std::mutex> l(m_);
                cv_.wait(l, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
                job = job_;
                jobs = jobs_;
            }
            if (k < jobs) (*job)(k);
            std::lock_guard<std::mutex> g(m_);
            if (--pending_ == 0) done_.notify_one();
        }
    }
    int nt_;
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    const std::function<void(int)>* job_ = nullptr;
    int jobs_ = 0;
    int pending_ = 0;
    unsigned long long gen_ = 0;
    bool stop_ = false;
};

struct tb_context {
    std::vector<DevState> devs;
    std::unique_ptr<HostPool> pool;  // staging copies (created on the first host-buffer solve)
    int mode = TB_MODE_EXACT;
    int fast_forward = 1;
    int form = TB_FORM_AUTO;
    int order = TB_ORDER_AUTO;
};

extern "C" {

const char* tb_last_error(void) { return g_err.c_str(); }
int64_t tb_kernel_launch_count(void) { return tbdev::launches(); }

void tb_config_default(tb_tron_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->tol_pg = 1e-6;
    c->max_iter = 200;
    c->cg_tol = 0.1;
    c->eta0 = 1e-4;
    c->sigma1 = 0.25;
    c->sigma2 = 0.5;
    c->sigma3 = 4.0;
    c->mu0 = 1e-2;
    c->mu1 = 1.0;
    c->interp_factor = 0.5;
    c->delta_max = 1e10;
}

// tron.hpp:70-80, same checks and messages
int tb_config_validate(const tb_tron_config* c) {
    if (!c) return set_err(TB_E_INVALID_ARGUMENT, "TronConfig: null");
    if (!(c->tol_pg > 0.0)) return set_err(TB_E_INVALID_ARGUMENT, "TronConfig: tol_pg must be > 0");
    if (c->has_delta0 && !(c->delta0 > 0.0))
        return set_err(TB_E_INVALID_ARGUMENT, "TronConfig: delta0 must be > 0");
    if (!(0.0 < c->sigma1 && c->sigma1 < c->sigma2 && c->sigma2 < 1.0 && 1.0 < c->sigma3))
        return set_err(TB_E_INVALID_ARGUMENT, "TronConfig: need 0 < sigma1 < sigma2 < 1 < sigma3");
    if (!(0.0 < c->eta0 && c->eta0 < 1.0)) return set_err(TB_E_INVALID_ARGUMENT, "TronConfig: need 0 < eta0 < 1");
    if (!(0.0 < c->mu0 && c->mu0 < 1.0)) return set_err(TB_E_INVALID_ARGUMENT, "TronConfig: need 0 < mu0 < 1");
    if (!(0.0 < c->interp_factor && c->interp_factor < 1.0))
        return set_err(TB_E_INVALID_ARGUMENT, "TronConfig: need 0 < interp_factor < 1");
    if (c->max_iter < 1) return set_err(TB_E_INVALID_ARGUMENT, "TronConfig: max_iter must be >= 1");
    return TB_OK;
}

int64_t tb_family_nparams(int32_t family, int32_t dim) {
    if (!tb_family_dim_ok(family, dim)) return -1;
    return tb_fam_nparams(family, dim);
}

int tb_context_create(const int32_t* devices, int32_t n_devices, tb_context** out) {
    if (!out) return set_err(TB_E_INVALID_ARGUMENT, "tb_context_create: null out");
    *out = nullptr;
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (n_devices < 1 || n_devices > 64)
        return set_err(TB_E_INVALID_ARGUMENT, "solve_batch: workers must be >= 1");
    tb_context* ctx = new tb_context;
    int prev = 0;
    cudaGetDevice(&prev);
    for (int k = 0; k < n_devices; ++k) {
        DevState d;
        d.device = devices ? devices[k] : k;
        if (d.device < 0 || d.device >= ndev) {
            tb_context_destroy(ctx);  // releases the devices set up so far
            return set_err(TB_E_INVALID_ARGUMENT, "tb_context_create: device %d out of range (%d visible)",
                           d.device, ndev);
        }
        cudaSetDevice(d.device);
        cudaError_t e = cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking);
        for (int i = 0; i < 8 && e == cudaSuccess; ++i) e = cudaStreamCreateWithFlags(&d.aux[i], cudaStreamNonBlocking);
        for (int i = 0; i < 4 && e == cudaSuccess; ++i) e = cudaEventCreate(&d.ev[i]);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d.fork, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d.join, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d.ws_ev, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d.ord_ev, cudaEventDisableTiming);
        if (e != cudaSuccess) {
            ctx->devs.push_back(d);  // the partially created streams / events are released with it
            tb_context_destroy(ctx);
            cudaSetDevice(prev);
            return set_err(TB_E_CUDA, "tb_context_create: %s", cudaGetErrorString(e));
        }
        ctx->devs.push_back(d);
    }
    cudaSetDevice(prev);
    *out = ctx;
    return TB_OK;
}

int tb_context_destroy(tb_context* ctx) {
    if (!ctx) return TB_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    for (auto& d : ctx->devs) {
        cudaSetDevice(d.device);
        if (d.stream) cudaStreamSynchronize(d.stream);
        for (auto& a : d.aux)
            if (a) cudaStreamSynchronize(a);
        for (auto& e : d.ev)
            if (e) cudaEventDestroy(e);
        if (d.fork) cudaEventDestroy(d.fork);
        if (d.join) cudaEventDestroy(d.join);
        if (d.ws_ev) cudaEventDestroy(d.ws_ev);
        if (d.ord_ev) cudaEventDestroy(d.ord_ev);
        if (d.stream) cudaStreamDestroy(d.stream);
        for (auto& a : d.aux)
            if (a) cudaStreamDestroy(a);
        d.in.release();
        d.out.release();
        d.flag.release();
        d.ws.release();
        d.hin.release();
        d.hout.release();
    }
    cudaSetDevice(prev);
    delete ctx;
    return TB_OK;
}

int tb_context_set_mode(tb_context* ctx, int32_t mode, int32_t fast_forward) {
    if (!ctx) return set_err(TB_E_INVALID_ARGUMENT, "null context");
    if (mode != TB_MODE_EXACT)
        return set_err(TB_E_INVALID_ARGUMENT, "only TB_MODE_EXACT is built in this version");
    ctx->mode = mode;
    if (fast_forward < 0 || fast_forward > 2) return set_err(TB_E_INVALID_ARGUMENT, "fast_forward must be 0, 1 or 2");
    ctx->fast_forward = fast_forward;
    return TB_OK;
}

int tb_host_alloc(int64_t bytes, void** out) {
    if (!out || bytes < 0) return set_err(TB_E_INVALID_ARGUMENT, "tb_host_alloc: bad arguments");
    *out = nullptr;
    if (bytes == 0) return TB_OK;
    CUDA_TRY(cudaHostAlloc(out, (size_t)bytes, cudaHostAllocPortable));
    return TB_OK;
}

int tb_host_free(void* p) {
    if (p) CUDA_TRY(cudaFreeHost(p));
    return TB_OK;
}

int tb_context_set_form(tb_context* ctx, int32_t form) {
    if (!ctx) return set_err(TB_E_INVALID_ARGUMENT, "null context");
    if (form != TB_FORM_AUTO && form != TB_FORM_WARP && form != TB_FORM_THREAD && form != TB_FORM_BLOCK)
        return set_err(TB_E_INVALID_ARGUMENT, "unknown kernel form %d", form);
    ctx->form = form;
    return TB_OK;
}

int tb_context_set_order(tb_context* ctx, int32_t order) {
    if (!ctx) return set_err(TB_E_INVALID_ARGUMENT, "null context");
    if (order != TB_ORDER_AUTO && order != TB_ORDER_INDEX && order != TB_ORDER_START_PG && order != TB_ORDER_CALLER)
        return set_err(TB_E_INVALID_ARGUMENT, "unknown launch order %d", order);
    ctx->order = order;
    return TB_OK;
}

int tb_imbalance(const double* times, int32_t n_iters, int32_t n_parts, double* nu, double* nu_max,
                 double* nu_min, double* nu_mean) {
    // batch.hpp:89-111
    if (n_iters < 1) return set_err(TB_E_INVALID_ARGUMENT, "imbalance: need at least one iteration");
    if (n_parts < 2) return set_err(TB_E_INVALID_ARGUMENT, "imbalance: need at least 2 partitions");
    for (int k = 0; k < n_iters; ++k) {
        double tmax = 0.0, tsum = 0.0;
        for (int p = 0; p < n_parts; ++p) {
            const double t = times[(long)k * n_parts + p];
            if (!(t > 0.0)) return set_err(TB_E_INVALID_ARGUMENT, "imbalance: partition times must be positive");
            tmax = std::max(tmax, t);
            tsum += t;
        }
        const double tmean = tsum / static_cast<double>(n_parts);
        nu[k] = (tmax / tmean - 1.0) * 100.0;
    }
    *nu_max = *std::max_element(nu, nu + n_iters);
    *nu_min = *std::min_element(nu, nu + n_iters);
    double s = 0.0;
    for (int k = 0; k < n_iters; ++k) s += nu[k];
    *nu_mean = s / static_cast<double>(n_iters);
    return TB_OK;
}

}  // extern "C"

namespace {

int check_batch(const tb_problem_batch* b, int64_t* nparams) {
    if (!b) return set_err(TB_E_INVALID_ARGUMENT, "solve_batch: null batch");
    if (b->count < 0) return set_err(TB_E_INVALID_ARGUMENT, "solve_batch: negative count");
    if (b->family < 0 || b->family >= TB_NUM_FAMILIES)
        return set_err(TB_E_INVALID_ARGUMENT, "solve_batch: unknown problem family %d", b->family);
    if (!tb_family_dim_ok(b->family, b->dim))
        return set_err(TB_E_INVALID_ARGUMENT, "solve_batch: dimension %d invalid for family %d", b->dim, b->family);
    if (b->dim > tbdev::max_dim())
        return set_err(TB_E_INVALID_ARGUMENT, "solve_batch: dimension %d exceeds device capacity %d", b->dim,
                       tbdev::max_dim());
    *nparams = tb_fam_nparams(b->family, b->dim);
    if (b->count > 0) {
        if (!b->x0 || !b->lower || !b->upper)
            return set_err(TB_E_INVALID_ARGUMENT, "solve_batch: null x0/lower/upper");
        if (*nparams > 0 && (!b->params || b->params_stride < *nparams))
            return set_err(TB_E_INVALID_ARGUMENT, "solve_batch: params missing or stride %lld < %lld",
                           (long long)b->params_stride, (long long)*nparams);
    }
    if (b->memspace != TB_MEM_HOST && b->memspace != TB_MEM_DEVICE)
        return set_err(TB_E_INVALID_ARGUMENT, "solve_batch: bad memspace");
    return TB_OK;
}

constexpr int64_t kChunkMin = 4096;  // problems per chunk of the host-buffer pipeline

// Debug builds only (-DTB_TRACE_HOST): host-side timeline of tb_solve_batch
// on stderr; `sync` waits for the device first (perturbs the overlap).
#ifdef TB_TRACE_HOST
#define TB_TRACE(what, sync)                                                                                  \
    do {                                                                                                     \
        if (sync) cudaDeviceSynchronize();                                                                    \
        fprintf(stderr, "[tb trace] %-22s %8.3f ms\n", what,                                                 \
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() * 1e3);         \
    } while (0)
#else
#define TB_TRACE(what, sync)
#endif

// Copy into page-locked staging with non-temporal stores: a DMA that reads
// lines the CPU just wrote (still dirty in its caches) runs at ~17 GB/s on
// the B200 boxes, the same bytes written with streaming stores at the full
// ~53 GB/s (scripts/micro/h2d_staging.cu), and the copy itself is faster.
void stream_memcpy(void* dst, const void* src, size_t bytes) {
#if defined(__SSE2__)
    char* d = static_cast<char*>(dst);
    const char* s = static_cast<const char*>(src);
    const size_t head = std::min(bytes, (size_t)((16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15));
    std::memcpy(d, s, head);
    size_t i = head;
    for (; i + 64 <= bytes; i += 64) {
        const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
        const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 16));
        const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 32));
        const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 48));
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), a);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 16), b);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 32), c);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 48), e);
    }
    _mm_sfence();
    std::memcpy(d + i, s + i, bytes - i);
#else
    std::memcpy(dst, src, bytes);
#endif
}

// Host copies between caller (pageable) memory and the pinned staging: one
// thread moves ~17 GB/s, so a set of copies of a few MB is split over host
// threads started once for the whole set (the staging of a ranked C2 batch is
// 28 MB in four arrays, 6 MB out in nine); `to_staging` selects the
// streaming stores.
struct HostCopy {
    void* dst;
    const void* src;
    size_t bytes;
};
void par_memcpy_set(HostPool* pool, const HostCopy* jobs, int njobs, bool to_staging) {
    constexpr size_t kPiece = size_t(1) << 18;
    size_t total = 0;
    for (int j = 0; j < njobs; ++j) total += jobs[j].src && jobs[j].dst ? jobs[j].bytes : 0;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t t = std::max<size_t>(1, std::min<size_t>(std::min<size_t>(hw, 8), total / kPiece));
    auto part = [&](size_t k) {  // slice k of every copy of the set
        for (int j = 0; j < njobs; ++j) {
            const HostCopy& c = jobs[j];
            if (!c.src || !c.dst) continue;
            const size_t a = c.bytes * k / t, b = c.bytes * (k + 1) / t;
            if (b <= a) continue;
            if (to_staging) stream_memcpy(static_cast<char*>(c.dst) + a, static_cast<const char*>(c.src) + a, b - a);
            else std::memcpy(static_cast<char*>(c.dst) + a, static_cast<const char*>(c.src) + a, b - a);
        }
    };
    if (t <= 1) {
        part(0);
        return;
    }
    if (pool) {
        const int tp = (int)std::min<size_t>(t, (size_t)pool->size());
        pool->run(tp, [&](int k) {
            for (size_t r = (size_t)k; r < t; r += (size_t)tp) part(r);
        });
        return;
    }
    std::vector<std::thread> th;
    th.reserve(t - 1);
    size_t k = 1;
    try {  // no exception may leave the C ABI: pieces without a thread are copied here
        for (; k < t; ++k) th.emplace_back(part, k);
    } catch (...) {
    }
    for (size_t r = k; r < t; ++r) part(r);
    part(0);
    for (auto& x : th) x.join();
}

// page-locked (or registered) host memory: async copies from pageable memory
// block the host, which would serialise the chunk pipeline
bool is_pinned(const void* p) {
    if (!p) return true;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}
// chunk counts (measured on C2 at 24 blocks/SM, 10-step bench): host-staged
// e2e 7.18 / 7.45 / 7.54 / 7.58 / 7.95 / 8.11 M solves/s at 1 / 2 / 3 / 4 / 6 /
// 8 chunks (smaller first H2D, finer copy/compute overlap); device-resident
// 8.32 / 8.65 / 8.34 / 8.25 / 8.28 / 8.41 ms -> 4.
#ifndef TB_HOST_CHUNKS
#define TB_HOST_CHUNKS 8  // experiments: rebuild with -DTB_HOST_CHUNKS=k (1..8; 1 disables the split)
#endif
#ifndef TB_DEVICE_CHUNKS
#define TB_DEVICE_CHUNKS 4
#endif
int64_t max_chunks(bool host) {
    const int64_t v = host ? TB_HOST_CHUNKS : TB_DEVICE_CHUNKS;
    return v < 1 ? 1 : (v > 8 ? 8 : v);  // one stream per chunk: aux[8]
}

struct OutPtrs {
    double *x_star, *f_star, *pg;
    int32_t *status, *iters;
    int64_t *cg, *fev, *flops;
    double* wall;
};

// carve result arrays for `cnt` problems of dim n out of one device buffer
size_t out_bytes(int64_t cnt, int n) {
    return (size_t)cnt * (sizeof(double) * (n + 3) + sizeof(int32_t) * 2 + sizeof(int64_t) * 3) + 256;
}
OutPtrs carve(void* base, int64_t cnt, int n) {
    char* p = static_cast<char*>(base);
    OutPtrs o;
    o.x_star = reinterpret_cast<double*>(p); p += sizeof(double) * cnt * n;
    o.f_star = reinterpret_cast<double*>(p); p += sizeof(double) * cnt;
    o.pg = reinterpret_cast<double*>(p); p += sizeof(double) * cnt;
    o.wall = reinterpret_cast<double*>(p); p += sizeof(double) * cnt;
    o.cg = reinterpret_cast<int64_t*>(p); p += sizeof(int64_t) * cnt;
    o.fev = reinterpret_cast<int64_t*>(p); p += sizeof(int64_t) * cnt;
    o.flops = reinterpret_cast<int64_t*>(p); p += sizeof(int64_t) * cnt;
    o.status = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * cnt;
    o.iters = reinterpret_cast<int32_t*>(p);
    return o;
}

const char* status_message(int st) {
    switch (st) {
        case TB_STATUS_EVALUATION_ERROR: return "EvaluationError: cauchy: non-finite quadratic model value";
        case TB_STATUS_ZERO_DIRECTION: return "invalid_argument: trqsol: direction is zero, no intersection";
        case TB_STATUS_SINGULAR_FACTOR: return "SingularFactorError: trtrs: zero diagonal";
        case TB_STATUS_INVALID_BOUNDS: return "invalid_argument: solve: lower bound exceeds upper bound";
    }
    return "unknown";
}

tbdev::KernelArgs make_args(const tb_problem_batch* b, int64_t np, const tb_tron_config* cfg, int ff, int form,
                            const double* x0, const double* lo, const double* up, const double* prm,
                            int64_t stride, int64_t cnt, const OutPtrs& o) {
    tbdev::KernelArgs a;
    a.n = b->dim;
    a.nparams = (int)np;
    a.count = cnt;
    a.stride = stride;
    a.x0 = x0;
    a.lo = lo;
    a.up = up;
    a.prm = np > 0 ? prm : nullptr;
    a.cfg = *cfg;
    a.fast_forward = ff;
    a.extrap = 1.0 / cfg->interp_factor;
    a.x_star = o.x_star;
    a.f_star = o.f_star;
    a.pg_norm = o.pg;
    a.status = o.status;
    a.iterations = o.iters;
    a.cg_iterations = o.cg;
    a.f_evals = o.fev;
    a.wall_time = o.wall;
    a.flops = o.flops;
    a.ws = nullptr;
    a.ws_bytes = 0;
    a.route_count = cnt;
    a.next = nullptr;
    a.form = form;
    a.skip = nullptr;
    a.order = nullptr;
    return a;
}

// attach the block kernel's workspace (d > 16), grown on demand; the launch
// on `st` is ordered after the previous workspace user (ws_ev)
cudaError_t attach_ws(DevState& d, int family, tbdev::KernelArgs& a, cudaStream_t st) {
    size_t need = 0;
    cudaError_t e = tbdev::tron_ws_need(family, a.n, a.count, a.form, &need);
    if (e != cudaSuccess || need == 0) return e;
    if ((e = d.ws.ensure(need)) != cudaSuccess) return e;
    a.ws = d.ws.p;
    a.ws_bytes = d.ws.cap;
    return cudaStreamWaitEvent(st, d.ws_ev, 0);
}
// after a launch that used the workspace
cudaError_t release_ws(DevState& d, const tbdev::KernelArgs& a, cudaStream_t st) {
    return a.ws ? cudaEventRecord(d.ws_ev, st) : cudaSuccess;
}

// Launch order (tron_order.cu).  AUTO ranks where the start
// projected-gradient norm was measured to predict the long solves
// (profiles/r02_order_ab.txt, device-resident, ms, index -> ranked): the
// branch family beyond one wave of warps (C2 7.39 -> 5.36; branch4 thread
// form x20,467 0.80 -> 0.74, x65,536 1.16 -> 0.90) and the d = 17..32 block
// kernel beyond one wave (ncvx32 x8,192 10.65 -> 9.45, ncvx24 7.10 -> 6.93).
// Elsewhere the ranking does not pay (ncvx d <= 16 and boxqp warp / thread
// forms, the d >= 33 block kernel: 0-17 % slower), so those keep index order.
bool want_order(int family, const tbdev::KernelArgs& a, int mode) {
    // counting runs are untimed; the order is 32-bit
    if (mode == TB_ORDER_INDEX || a.count < 2 || a.flops || a.count > 0x7fffffffLL) return false;
    if (mode == TB_ORDER_START_PG) return true;
    const long long wave = 32LL * tbdev::device_sm_count();
    const int form = tbdev::tron_form(family, a);
    if (family == TB_FAMILY_BRANCH) return form == TB_FORM_THREAD ? a.count >= 16384 : a.count > wave;
    return form == TB_FORM_BLOCK && a.n >= 17 && a.n <= 32 && a.count > 16LL * tbdev::device_sm_count();
}
// rank the launch's problems into the device's order workspace on `st`
// (ordered after the previous user of that workspace, like attach_ws)
cudaError_t attach_order(DevState& d, int family, tbdev::KernelArgs& a, int mode, cudaStream_t st) {
    a.order = nullptr;
    if (!want_order(family, a, mode)) return cudaSuccess;
    cudaError_t e = d.ord.ensure(tbdev::order_ws_bytes(a.count));
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, d.ord_ev, 0);
    if (e == cudaSuccess) e = tbdev::launch_order(family, a, d.ord.p, st, &a.order);
    return e;
}
// ranked launches, and TB_ORDER_CALLER (the caller sorted the batch), run as
// one launch in order
bool one_launch(const tbdev::KernelArgs& a, int mode) { return a.order || mode == TB_ORDER_CALLER; }
cudaError_t release_order(DevState& d, const tbdev::KernelArgs& a, cudaStream_t st) {
    return a.order ? cudaEventRecord(d.ord_ev, st) : cudaSuccess;
}

// Device-resident batch on the warp kernel: `nch` concurrent chunk launches
// forked from `st` onto the device's chunk streams and joined back, so the
// long-running problems of one chunk overlap the bulk of the others (the
// launch finishes with its slowest problem).
cudaError_t launch_split(DevState& d, int family, const tbdev::KernelArgs& a, cudaStream_t st, int nch) {
    if (nch <= 1) return tbdev::launch_tron(family, a, st);
    cudaError_t e = cudaEventRecord(d.fork, st);
    for (int k = 0; k < nch && e == cudaSuccess; ++k) e = cudaStreamWaitEvent(d.aux[k], d.fork, 0);
    for (int k = 0; k < nch && e == cudaSuccess; ++k) {
        const int64_t a0 = a.count * k / nch, a1 = a.count * (k + 1) / nch;
        tbdev::KernelArgs c = a;
        const int n = a.n;
        c.count = a1 - a0;
        if (c.order) {  // ranked: chunk k takes launch slots [a0, a1) of the whole batch
            c.order += a0;
            e = tbdev::launch_tron(family, c, d.aux[k]);
            continue;
        }
        c.x0 += a0 * n;
        c.lo += a0 * n;
        c.up += a0 * n;
        if (c.prm) c.prm += a0 * a.stride;
        if (c.x_star) c.x_star += a0 * n;
        if (c.f_star) c.f_star += a0;
        if (c.pg_norm) c.pg_norm += a0;
        if (c.status) c.status += a0;
        if (c.iterations) c.iterations += a0;
        if (c.cg_iterations) c.cg_iterations += a0;
        if (c.f_evals) c.f_evals += a0;
        if (c.wall_time) c.wall_time += a0;
        if (c.flops) c.flops += a0;
        e = tbdev::launch_tron(family, c, d.aux[k]);
    }
    for (int k = 0; k < nch && e == cudaSuccess; ++k) {
        e = cudaEventRecord(d.join, d.aux[k]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, d.join, 0);
    }
    return e;
}

// chunk count of a device-resident batch: only the one-shot warp kernel is
// split (the persistent forms refill their groups from one counter; the
// block kernel owns one workspace per device)
int device_chunks(const tbdev::KernelArgs& a, int family) {
    if (tbdev::tron_form(family, a) != TB_FORM_WARP) return 1;
    return a.count >= 2 * kChunkMin ? (int)std::min<int64_t>(max_chunks(false), a.count / kChunkMin) : 1;
}

}  // namespace

extern "C" int tb_solve_batch_async(tb_context* ctx, const tb_problem_batch* b, const tb_tron_config* cfg,
                                    tb_batch_result* r, void* stream) {
    if (!ctx || !r) return set_err(TB_E_INVALID_ARGUMENT, "solve_batch: null context/result");
    int rc = tb_config_validate(cfg);
    if (rc) return rc;
    int64_t np = 0;
    if ((rc = check_batch(b, &np))) return rc;
    if (ctx->devs.size() != 1 || b->memspace != TB_MEM_DEVICE || r->memspace != TB_MEM_DEVICE)
        return set_err(TB_E_INVALID_ARGUMENT, "solve_batch_async: needs a 1-device context and device memory");
    DevState& d = ctx->devs[0];
    int prev = 0;
    cudaGetDevice(&prev);
    CUDA_TRY(cudaSetDevice(d.device));
    struct Restore {
        int dev;
        ~Restore() { cudaSetDevice(dev); }
    } restore{prev};  // the caller's current device is left as it was
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d.stream;
    OutPtrs o{r->x_star, r->f_star, r->pg_norm, r->status, r->iterations, r->cg_iterations, r->f_evals, r->flops,
              r->wall_time};
    tbdev::KernelArgs a = make_args(b, np, cfg, ctx->fast_forward, ctx->form, b->x0, b->lower, b->upper, b->params,
                                    b->params_stride, b->count, o);
    CUDA_TRY(attach_ws(d, b->family, a, st));
    CUDA_TRY(attach_order(d, b->family, a, ctx->order, st));
    CUDA_TRY(launch_split(d, b->family, a, st, one_launch(a, ctx->order) ? 1 : device_chunks(a, b->family)));
    CUDA_TRY(release_order(d, a, st));
    CUDA_TRY(release_ws(d, a, st));
    return TB_OK;
}

// tb_solve_batch_packed's callbacks (null for tb_solve_batch)
struct HostCb {
    tb_pack_fn pack;
    tb_unpack_fn unpack;
    void* user;
};

static int solve_batch_impl(tb_context* ctx, const tb_problem_batch* b, const tb_tron_config* cfg,
                            tb_batch_result* r, const HostCb* cb) {
    using clock = std::chrono::steady_clock;
    if (!ctx || !r) return set_err(TB_E_INVALID_ARGUMENT, "solve_batch: null context/result");
    int rc = tb_config_validate(cfg);
    if (rc) return rc;
    int64_t np = 0;
    if ((rc = check_batch(b, &np))) return rc;
    const int G = (int)ctx->devs.size();
    if ((b->memspace == TB_MEM_DEVICE || r->memspace == TB_MEM_DEVICE) && G != 1)
        return set_err(TB_E_INVALID_ARGUMENT, "solve_batch: device-resident buffers need a 1-device context");
    const int n = b->dim;
    const int64_t N = b->count;
    const int64_t stride = np > 0 ? b->params_stride : 0;
    const bool in_host = b->memspace == TB_MEM_HOST;
    const bool out_host = r->memspace == TB_MEM_HOST;
    int prev = 0;
    cudaGetDevice(&prev);
    struct Restore {
        int dev;
        ~Restore() { cudaSetDevice(dev); }
    } restore{prev};  // every return path leaves the caller's device current
    const auto t0 = clock::now();

    r->n_partitions = G;
    std::vector<int64_t> lo(G), cnt(G);
    {
        const int64_t base = N / G, rem = N % G;  // batch.hpp:61-70
        int64_t s = 0;
        for (int k = 0; k < G; ++k) {
            lo[k] = s;
            cnt[k] = base + (k < rem ? 1 : 0);
            s += cnt[k];
        }
    }

    // Host buffers: the partition is cut into chunks, each on its own stream,
    // so the H2D copy of chunk i+1 and the D2H copy of chunk i-1 overlap the
    // solves, and a long-running problem in one chunk never holds back the
    // next chunk (warp / thread kernels; the persistent block kernel owns one
    // workspace per device and runs unchunked).  Page-locked caller buffers
    // are copied directly; pageable ones (e.g. the C++ drop-in's vectors) go
    // through library-owned pinned staging: the host copies chunk i+1's inputs
    // into it while chunk i solves, and copies chunk i's results out while
    // later chunks solve.
    // callbacks: the caller packs into / unpacks from the pinned staging
    const bool in_pinned = !cb && (!in_host || (is_pinned(b->x0) && is_pinned(b->lower) && is_pinned(b->upper) &&
                                                (np == 0 || is_pinned(b->params))));
    const bool out_pinned =
        !cb && (!out_host || (is_pinned(r->x_star) && is_pinned(r->f_star) && is_pinned(r->pg_norm) &&
                              is_pinned(r->status) && is_pinned(r->iterations) && is_pinned(r->cg_iterations) &&
                              is_pinned(r->f_evals) && is_pinned(r->wall_time) && is_pinned(r->flops)));
    if (((in_host && !in_pinned) || (out_host && !out_pinned)) && !ctx->pool) {
        try {  // host threads for the staging copies; without them the copies run serially
            ctx->pool = std::make_unique<HostPool>((int)std::min(8u, std::max(1u, std::thread::hardware_concurrency())));
        } catch (...) {
        }
    }
    int64_t first_bad = -1;  // first problem the reference would have thrown on (batch.hpp:75-76)
    int bad_status = 0;
    std::vector<int> nchs(G, 1);
    std::vector<char> rankeds(G, 0);
    for (int k = 0; k < G; ++k) {
        DevState& d = ctx->devs[k];
        CUDA_TRY(cudaSetDevice(d.device));
        const int64_t c = cnt[k];
        CUDA_TRY(cudaEventRecord(d.ev[0], d.stream));
        const bool staged = (in_host || out_host) && c > 0;  // the host-buffer pipeline
        const bool in_stage = in_host && !in_pinned && c > 0;
        const bool out_stage = out_host && !out_pinned && c > 0;
        size_t ws_need = 0;  // > 0: the persistent block kernel (one workspace per device): no chunking
        CUDA_TRY(tbdev::tron_ws_need(b->family, n, c, ctx->form, &ws_need));
        // Ranked partitions solve in ONE launch in rank order
        // once the whole partition is on the device (a problem's rank spans
        // the partition): page-locked inputs go over in one piece; pageable
        // inputs and the callers' pack callbacks keep the chunks, so the host
        // staging (context thread team, streaming stores) or packing of chunk
        // i+1 overlaps chunk i's transfer
        bool ranked = false;
        if (staged) {
            tbdev::KernelArgs stub = make_args(b, np, cfg, ctx->fast_forward, ctx->form, nullptr, nullptr, nullptr,
                                               nullptr, stride, c, OutPtrs{});
            stub.flops = r->flops;  // a counting run is never ranked
            stub.route_count = c;
            ranked = want_order(b->family, stub, ctx->order) || ctx->order == TB_ORDER_CALLER;
        }
        const int nch = (staged && ws_need == 0 && c >= 2 * kChunkMin && (!ranked || cb || in_stage))
                            ? (int)std::min<int64_t>(max_chunks(true), c / kChunkMin)
                            : 1;
        nchs[k] = nch;
        if (nch > 1) {
            CUDA_TRY(cudaEventRecord(d.fork, d.stream));
            for (int ch = 0; ch < nch; ++ch) CUDA_TRY(cudaStreamWaitEvent(d.aux[ch], d.fork, 0));
        }
        const size_t vb = sizeof(double) * (size_t)c * n;
        const size_t pb = sizeof(double) * (size_t)c * stride;
        char* inp = nullptr;
        char* hinp = nullptr;
        if (in_host && c > 0) {
            CUDA_TRY(d.in.ensure(3 * vb + pb + 64));
            inp = static_cast<char*>(d.in.p);
            if (in_stage) {
                CUDA_TRY(d.hin.ensure(3 * vb + pb + 64));
                hinp = static_cast<char*>(d.hin.p);
            }
        }
        OutPtrs hst{};  // pinned output staging (pageable outputs)
        if (out_stage) {
            CUDA_TRY(d.hout.ensure(out_bytes(c, n)));
            hst = carve(d.hout.p, c, n);
        }
        OutPtrs ofull;
        if (out_host) {
            CUDA_TRY(d.out.ensure(out_bytes(c, n)));
            ofull = carve(d.out.p, c, n);
            if (!r->flops) ofull.flops = nullptr;  // non-null flops selects the counting kernel variant
        } else {
            ofull = OutPtrs{r->x_star, r->f_star, r->pg_norm, r->status, r->iterations, r->cg_iterations,
                            r->f_evals, r->flops, r->wall_time};
            // status is needed for the error scan even if the caller skips it
            if (!ofull.status) {
                CUDA_TRY(d.out.ensure(out_bytes(c, n)));
                ofull.status = carve(d.out.p, c, n).status;
            }
        }
        // the whole partition's launch arguments (device copies of the inputs)
        auto part_args = [&]() {
            const double *x0, *lw, *up, *prm;
            if (in_host) {
                x0 = reinterpret_cast<const double*>(inp);
                lw = reinterpret_cast<const double*>(inp + vb);
                up = reinterpret_cast<const double*>(inp + 2 * vb);
                prm = pb ? reinterpret_cast<const double*>(inp + 3 * vb) : nullptr;
            } else {
                x0 = b->x0 + lo[k] * n;
                lw = b->lower + lo[k] * n;
                up = b->upper + lo[k] * n;
                prm = np > 0 ? b->params + lo[k] * stride : nullptr;
            }
            tbdev::KernelArgs a = make_args(b, np, cfg, ctx->fast_forward, ctx->form, x0, lw, up, prm, stride, c, ofull);
            a.route_count = c;
            return a;
        };
        rankeds[k] = ranked;
        for (int ch = 0; ch < nch; ++ch) {
            cudaStream_t st = nch > 1 ? d.aux[ch] : d.stream;
            const int64_t a0 = c * ch / nch, a1 = c * (ch + 1) / nch, cc = a1 - a0;  // local range
            const int64_t g0 = lo[k] + a0;                                             // global index
            const double *x0 = cb ? nullptr : b->x0 + g0 * n, *lw = cb ? nullptr : b->lower + g0 * n,
                         *up = cb ? nullptr : b->upper + g0 * n;
            const double* prm = (np > 0 && !cb) ? b->params + g0 * stride : nullptr;
            if (in_host && cc > 0) {
                const size_t cvb = sizeof(double) * (size_t)cc * n, cpb = sizeof(double) * (size_t)cc * stride;
                char* dx = inp + sizeof(double) * (size_t)a0 * n;
                char* dl = inp + vb + sizeof(double) * (size_t)a0 * n;
                char* du = inp + 2 * vb + sizeof(double) * (size_t)a0 * n;
                char* dp = inp + 3 * vb + sizeof(double) * (size_t)a0 * stride;
                if (in_stage) {  // pageable -> pinned staging (host copy), then an async H2D from it
                    char* hx = hinp + (dx - inp);
                    char* hl = hinp + (dl - inp);
                    char* hu = hinp + (du - inp);
                    char* hp = hinp + (dp - inp);
                    if (cb) {
                        cb->pack(cb->user, g0, g0 + cc, reinterpret_cast<double*>(hx), reinterpret_cast<double*>(hl),
                                 reinterpret_cast<double*>(hu), cpb ? reinterpret_cast<double*>(hp) : nullptr);
                    } else {
                        const HostCopy set[4] = {{hx, x0, cvb}, {hl, lw, cvb}, {hu, up, cvb}, {hp, prm, cpb}};
                        par_memcpy_set(ctx->pool.get(), set, 4, true);
                    }
                    x0 = reinterpret_cast<const double*>(hx);
                    lw = reinterpret_cast<const double*>(hl);
                    up = reinterpret_cast<const double*>(hu);
                    prm = cpb ? reinterpret_cast<const double*>(hp) : nullptr;
                }
                CUDA_TRY(cudaMemcpyAsync(dx, x0, cvb, cudaMemcpyHostToDevice, st));
                CUDA_TRY(cudaMemcpyAsync(dl, lw, cvb, cudaMemcpyHostToDevice, st));
                CUDA_TRY(cudaMemcpyAsync(du, up, cvb, cudaMemcpyHostToDevice, st));
                if (cpb) CUDA_TRY(cudaMemcpyAsync(dp, prm, cpb, cudaMemcpyHostToDevice, st));
                x0 = reinterpret_cast<const double*>(dx);
                lw = reinterpret_cast<const double*>(dl);
                up = reinterpret_cast<const double*>(du);
                prm = cpb ? reinterpret_cast<const double*>(dp) : nullptr;
            }
            if (ranked) continue;  // inputs only; the ranked launch follows the loop
            auto off = [&](auto* p, int64_t m) { return p ? p + a0 * m : p; };
            OutPtrs o{off(ofull.x_star, n), off(ofull.f_star, 1), off(ofull.pg, 1), off(ofull.status, 1),
                      off(ofull.iters, 1), off(ofull.cg, 1),    off(ofull.fev, 1), off(ofull.flops, 1),
                      off(ofull.wall, 1)};
            tbdev::KernelArgs a = make_args(b, np, cfg, ctx->fast_forward, ctx->form, x0, lw, up, prm, stride, cc, o);
            a.route_count = c;  // kernel-form routing by the partition, not the pipeline chunk
            CUDA_TRY(attach_ws(d, b->family, a, st));
            if (ch == 0) CUDA_TRY(cudaEventRecord(d.ev[1], st));
            if (!staged) {
                CUDA_TRY(attach_order(d, b->family, a, ctx->order, st));
                // ranked: one launch in rank order (concurrent chunk launches
                // would interleave their dispatch and blur the order)
                CUDA_TRY(launch_split(d, b->family, a, st, one_launch(a, ctx->order) ? 1 : device_chunks(a, b->family)));
                CUDA_TRY(release_order(d, a, st));
            } else {
                CUDA_TRY(tbdev::launch_tron(b->family, a, st));
            }
            CUDA_TRY(release_ws(d, a, st));
            if (ch == nch - 1 && nch == 1) CUDA_TRY(cudaEventRecord(d.ev[2], st));
            if (out_host && cc > 0) {
                // pinned caller buffers: straight into them; pageable: into
                // the pinned staging (copied out after the chunk completes)
                auto tgt = [&](auto* user, auto* stage, int64_t m) -> decltype(user) {
                    if (!user && !(cb && stage)) return nullptr;  // callbacks: every report field
                    return out_stage ? stage + a0 * m : user + g0 * m;
                };
                auto cp = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
                    if (!dst || !src) return cudaSuccess;
                    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st);
                };
                CUDA_TRY(cp(tgt(r->x_star, hst.x_star, n), o.x_star, sizeof(double) * cc * n));
                CUDA_TRY(cp(tgt(r->f_star, hst.f_star, 1), o.f_star, sizeof(double) * cc));
                CUDA_TRY(cp(tgt(r->pg_norm, hst.pg, 1), o.pg, sizeof(double) * cc));
                CUDA_TRY(cp(tgt(r->status, hst.status, 1), o.status, sizeof(int32_t) * cc));
                CUDA_TRY(cp(tgt(r->iterations, hst.iters, 1), o.iters, sizeof(int32_t) * cc));
                CUDA_TRY(cp(tgt(r->cg_iterations, hst.cg, 1), o.cg, sizeof(int64_t) * cc));
                CUDA_TRY(cp(tgt(r->f_evals, hst.fev, 1), o.fev, sizeof(int64_t) * cc));
                CUDA_TRY(cp(tgt(r->flops, hst.flops, 1), o.flops, sizeof(int64_t) * cc));
                CUDA_TRY(cp(tgt(r->wall_time, hst.wall, 1), o.wall, sizeof(double) * cc));
            }
        }
        if (nch > 1) {  // join the chunk streams back into the partition's stream
            for (int ch = 0; ch < nch; ++ch) {
                CUDA_TRY(cudaEventRecord(d.join, d.aux[ch]));
                CUDA_TRY(cudaStreamWaitEvent(d.stream, d.join, 0));
            }
            if (!ranked) CUDA_TRY(cudaEventRecord(d.ev[2], d.stream));  // chunked: includes the last D2H
        }
        TB_TRACE("inputs issued", false);
        TB_TRACE("inputs on device", true);
        if (ranked) {
            tbdev::KernelArgs a = part_args();
            CUDA_TRY(attach_ws(d, b->family, a, d.stream));
            CUDA_TRY(cudaEventRecord(d.ev[1], d.stream));
            CUDA_TRY(attach_order(d, b->family, a, ctx->order, d.stream));
            CUDA_TRY(tbdev::launch_tron(b->family, a, d.stream));
            CUDA_TRY(release_order(d, a, d.stream));
            CUDA_TRY(release_ws(d, a, d.stream));
            CUDA_TRY(cudaEventRecord(d.ev[2], d.stream));
            TB_TRACE("ranked solve done", true);
            if (out_host) {
                auto tgt = [&](auto* user, auto* stage, int64_t m) -> decltype(user) {
                    if (!user && !(cb && stage)) return nullptr;  // callbacks: every report field
                    return out_stage ? stage : user + lo[k] * m;
                };
                auto cp = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
                    if (!dst || !src) return cudaSuccess;
                    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, d.stream);
                };
                const OutPtrs& o = ofull;
                CUDA_TRY(cp(tgt(r->x_star, hst.x_star, n), o.x_star, sizeof(double) * c * n));
                CUDA_TRY(cp(tgt(r->f_star, hst.f_star, 1), o.f_star, sizeof(double) * c));
                CUDA_TRY(cp(tgt(r->pg_norm, hst.pg, 1), o.pg, sizeof(double) * c));
                CUDA_TRY(cp(tgt(r->status, hst.status, 1), o.status, sizeof(int32_t) * c));
                CUDA_TRY(cp(tgt(r->iterations, hst.iters, 1), o.iters, sizeof(int32_t) * c));
                CUDA_TRY(cp(tgt(r->cg_iterations, hst.cg, 1), o.cg, sizeof(int64_t) * c));
                CUDA_TRY(cp(tgt(r->f_evals, hst.fev, 1), o.fev, sizeof(int64_t) * c));
                CUDA_TRY(cp(tgt(r->flops, hst.flops, 1), o.flops, sizeof(int64_t) * c));
                CUDA_TRY(cp(tgt(r->wall_time, hst.wall, 1), o.wall, sizeof(double) * c));
            }
        }
        CUDA_TRY(cudaEventRecord(d.ev[3], d.stream));
    }

    TB_TRACE("all issued", false);
    TB_TRACE("results on host", true);
    // pageable outputs: copy each chunk out of the pinned staging as soon as
    // it completes (later chunks keep solving meanwhile)
    if (out_host && !out_pinned) {
        for (int k = 0; k < G; ++k) {
            DevState& d = ctx->devs[k];
            const int64_t c = cnt[k];
            if (c == 0) continue;
            CUDA_TRY(cudaSetDevice(d.device));
            const OutPtrs hst = carve(d.hout.p, c, n);
            const int nch = nchs[k];
            for (int ch = 0; ch < nch; ++ch) {
                // ranked: every result arrives with the partition's one D2H
                CUDA_TRY(cudaStreamSynchronize(nch > 1 && !rankeds[k] ? d.aux[ch] : d.stream));
                const int64_t a0 = c * ch / nch, a1 = c * (ch + 1) / nch, cc = a1 - a0, g0 = lo[k] + a0;
                if (cb) {  // the chunk's reports, straight from the staging
                    for (int64_t i = 0; i < cc && first_bad < 0; ++i)
                        if (hst.status[a0 + i] >= TB_STATUS_EVALUATION_ERROR) {
                            first_bad = g0 + i;
                            bad_status = hst.status[a0 + i];
                        }
                    tb_batch_result v{};
                    v.x_star = hst.x_star + a0 * n;
                    v.f_star = hst.f_star + a0;
                    v.pg_norm = hst.pg + a0;
                    v.status = hst.status + a0;
                    v.iterations = hst.iters + a0;
                    v.cg_iterations = hst.cg + a0;
                    v.f_evals = hst.fev + a0;
                    v.wall_time = hst.wall + a0;
                    v.memspace = TB_MEM_HOST;
                    if (cc > 0) cb->unpack(cb->user, g0, g0 + cc, &v);
                    continue;
                }
                HostCopy set[9];
                int nj = 0;
                auto out = [&](auto* user, auto* stage, int64_t m) {
                    if (user) set[nj++] = {user + g0 * m, stage + a0 * m, sizeof(*user) * (size_t)(cc * m)};
                };
                out(r->x_star, hst.x_star, n);
                out(r->f_star, hst.f_star, 1);
                out(r->pg_norm, hst.pg, 1);
                out(r->status, hst.status, 1);
                out(r->iterations, hst.iters, 1);
                out(r->cg_iterations, hst.cg, 1);
                out(r->f_evals, hst.fev, 1);
                out(r->flops, hst.flops, 1);
                out(r->wall_time, hst.wall, 1);
                par_memcpy_set(ctx->pool.get(), set, nj, false);
            }
        }
    }
    TB_TRACE("copied out", false);
    double kmax = 0.0;
    for (int k = 0; k < G; ++k) {
        DevState& d = ctx->devs[k];
        CUDA_TRY(cudaSetDevice(d.device));
        CUDA_TRY(cudaStreamSynchronize(d.stream));
        float ms_part = 0.f, ms_kern = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms_part, d.ev[0], d.ev[3]));
        CUDA_TRY(cudaEventElapsedTime(&ms_kern, d.ev[1], d.ev[2]));
        if (k < 64) r->partition_times[k] = 1e-3 * ms_part;
        kmax = std::max(kmax, 1e-3 * (double)ms_kern);
    }
    r->kernel_time = kmax;
    r->batch_wall_time = std::chrono::duration<double>(clock::now() - t0).count();

    // batch.hpp:75-76: the first problem (input order) the reference would
    // have thrown on turns the whole call into an error (callbacks: found
    // while unpacking).
    for (int k = 0; k < G && first_bad < 0 && !cb; ++k) {
        const int64_t c = cnt[k];
        if (c == 0) continue;
        DevState& d = ctx->devs[k];
        cudaSetDevice(d.device);
        const int32_t* st_dev = nullptr;
        if (out_host && r->status) {
            for (int64_t i = 0; i < c; ++i)
                if (r->status[lo[k] + i] >= TB_STATUS_EVALUATION_ERROR) {
                    first_bad = lo[k] + i;
                    bad_status = r->status[lo[k] + i];
                    break;
                }
            continue;
        }
        st_dev = out_host ? carve(d.out.p, c, n).status : (r->status ? r->status : carve(d.out.p, c, n).status);
        CUDA_TRY(d.flag.ensure(sizeof(unsigned long long)));
        const unsigned long long init = ~0ull;
        CUDA_TRY(cudaMemcpyAsync(d.flag.p, &init, sizeof init, cudaMemcpyHostToDevice, d.stream));
        first_error_kernel<<<(unsigned)((c + 255) / 256), 256, 0, d.stream>>>(
            st_dev, c, static_cast<unsigned long long*>(d.flag.p));
        CUDA_TRY(cudaGetLastError());
        tbdev::note_launches(1);
        unsigned long long idx = ~0ull;
        CUDA_TRY(cudaMemcpyAsync(&idx, d.flag.p, sizeof idx, cudaMemcpyDeviceToHost, d.stream));
        CUDA_TRY(cudaStreamSynchronize(d.stream));
        if (idx != ~0ull) {
            int32_t s = 0;
            CUDA_TRY(cudaMemcpy(&s, st_dev + idx, sizeof s, cudaMemcpyDeviceToHost));
            first_bad = lo[k] + (int64_t)idx;
            bad_status = s;
        }
    }
    if (first_bad >= 0)
        return set_err(TB_E_PROBLEM, "problem %lld: %s", (long long)first_bad, status_message(bad_status));
    return TB_OK;
}

extern "C" int tb_solve_batch(tb_context* ctx, const tb_problem_batch* b, const tb_tron_config* cfg,
                              tb_batch_result* r) {
    return solve_batch_impl(ctx, b, cfg, r, nullptr);
}

extern "C" int tb_solve_batch_packed(tb_context* ctx, int32_t family, int32_t dim, int64_t count,
                                     const tb_tron_config* cfg, tb_pack_fn pack, tb_unpack_fn unpack, void* user,
                                     tb_batch_result* r) {
    if (!pack || !unpack) return set_err(TB_E_INVALID_ARGUMENT, "solve_batch_packed: null pack/unpack callback");
    if (!r) return set_err(TB_E_INVALID_ARGUMENT, "solve_batch: null context/result");
    // the batch's arrays are never read (the callbacks fill the staging);
    // non-null placeholders satisfy the argument checks
    static double placeholder;
    tb_problem_batch b{family, dim, count, &placeholder, &placeholder, &placeholder, &placeholder,
                       tb_family_nparams(family, dim) > 0 ? tb_family_nparams(family, dim) : 0, TB_MEM_HOST};
    tb_batch_result agg{};
    agg.memspace = TB_MEM_HOST;
    const HostCb cb{pack, unpack, user};
    const int rc = solve_batch_impl(ctx, &b, cfg, &agg, &cb);
    std::memcpy(r->partition_times, agg.partition_times, sizeof agg.partition_times);
    r->n_partitions = agg.n_partitions;
    r->batch_wall_time = agg.batch_wall_time;
    r->kernel_time = agg.kernel_time;
    return rc;
}
