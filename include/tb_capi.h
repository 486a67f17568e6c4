/*
 * tb_capi.h — C ABI of the B200 batched TRON solver (libtronbatch_b200.so).
 *
 * This is the drop-in boundary for the reference's solver path.  The
 * reference (`/root/reference/proj/include/tronbatch/`) is a header-only C++20
 * library whose API is C++ templates, not an FFI; every entry point below
 * replaces one reference interface, cited file:line.  The C++ mirror
 * `include/tronbatch_gpu/solve_batch.hpp` re-exposes exactly the reference
 * types and signatures on top of this ABI.
 *
 * Conventions: plain pointers and sizes only, no CUDA/torch types in the
 * signatures (streams travel as void*).  Functions return TB_OK or an error
 * code; tb_last_error() returns a thread-local message.  Batch arrays are
 * problem-major: x0/lower/upper/x_star are [count][dim], params is
 * [count][params_stride].
 */
#ifndef TB_CAPI_H
#define TB_CAPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes ------------------------------------------------------ */
#define TB_OK 0
#define TB_E_INVALID_ARGUMENT 1 /* std::invalid_argument in the reference */
#define TB_E_CUDA 2
#define TB_E_NCCL 3
#define TB_E_PROBLEM 4 /* a problem raised what the reference would throw; see statuses */

/* ---- per-problem status (tron.hpp:83 SolveStatus + extensions) ---------- */
#define TB_STATUS_CONVERGED 0            /* SolveStatus::Converged */
#define TB_STATUS_ITER_LIMIT 1           /* SolveStatus::IterLimit */
#define TB_STATUS_FACTORIZATION_FAILED 2 /* SolveStatus::FactorizationFailed */
/* extensions: where the reference throws out of solve() (tron.hpp:192,
 * dense.hpp:222, tron.hpp:170, tron.hpp:466) the device records a status and
 * the host wrappers rethrow the reference exception type. */
#define TB_STATUS_EVALUATION_ERROR 3 /* EvaluationError, tron.hpp:192 */
#define TB_STATUS_ZERO_DIRECTION 4   /* invalid_argument from trqsol, tron.hpp:170 */
#define TB_STATUS_SINGULAR_FACTOR 5  /* SingularFactorError, dense.hpp:222 */
#define TB_STATUS_INVALID_BOUNDS 6   /* invalid_argument, tron.hpp:465-466 */

/* ---- problem families (tron.hpp:28-36 BoundedProblem callbacks become
 *      compile-time device families; see csrc/tb_families.h) ------------- */
#define TB_FAMILY_HS45 0   /* batch.hpp:116-173 Hs45Problem */
#define TB_FAMILY_BOXQP 1  /* tests/support/boxqp_oracle.hpp:44-62 make_quadratic */
#define TB_FAMILY_NCVX 2   /* synthetic nonconvex family */
#define TB_FAMILY_BRANCH 3 /* ADMM branch subproblem Eq.(3), dim 4 or 6 (line limits) */

#define TB_MEM_HOST 0
#define TB_MEM_DEVICE 1

#define TB_MODE_EXACT 0 /* reference op order, no FMA: bitwise parity (the only mode) */

/* Kernel form of a batch (tb_context_set_form).  Every form computes the same
 * bits; the form only changes speed.  AUTO routes by family, dimension and
 * batch size; the others force a form where it exists for the
 * dimension (otherwise AUTO's choice is used). */
#define TB_FORM_AUTO 0
#define TB_FORM_WARP 1   /* one warp per problem, d <= 32 */
#define TB_FORM_THREAD 3 /* one thread per problem, d = 4 */
#define TB_FORM_BLOCK 4  /* 32 / 64 / 128 threads per problem, persistent, d >= 9 */

/* Launch order of a batch (tb_context_set_order).  Results never depend on
 * it (each problem is solved independently and reported at its own index);
 * it decides which problems start first.  START_PG launches the problems in
 * descending projected-gradient norm at their clipped start points, the
 * quantity solve() tests first and a good predictor of the iterations a
 * problem needs, so the long solves start early instead of forming the
 * launch's tail.  AUTO uses it where it was measured to pay
 * (one-warp-per-problem launches larger than one wave), INDEX never. */
#define TB_ORDER_AUTO 0
#define TB_ORDER_INDEX 1
#define TB_ORDER_START_PG 2
/* the caller's own order (a batch it sorted by its own cost estimate), as
 * ONE launch: problem k starts k-th */
#define TB_ORDER_CALLER 3

/* TronConfig (tron.hpp:54-81), field for field; std::optional delta0 becomes
 * has_delta0 + delta0. */
typedef struct tb_tron_config {
    double tol_pg;
    int32_t has_delta0;
    double delta0;
    int32_t max_iter;
    double cg_tol;
    double eta0;
    double sigma1;
    double sigma2;
    double sigma3;
    double mu0;
    double mu1;
    double interp_factor;
    double delta_max;
} tb_tron_config;

/* std::vector<P> problems + std::vector<Vector> x0s of solve_batch
 * (batch.hpp:27-29): a family id, the bounds of each problem
 * (BoundedProblem::lower/upper, tron.hpp:31-32) and its parameters. */
typedef struct tb_problem_batch {
    int32_t family;
    int32_t dim;
    int64_t count;
    const double* x0;     /* [count][dim] */
    const double* lower;  /* [count][dim], -inf allowed (tron.hpp:17) */
    const double* upper;  /* [count][dim], +inf allowed */
    const double* params; /* [count][params_stride], may be NULL for HS45 */
    int64_t params_stride;
    int32_t memspace; /* TB_MEM_HOST or TB_MEM_DEVICE for all five arrays */
} tb_problem_batch;

/* BatchResult (batch.hpp:17-22) of SolveReport (tron.hpp:94-103) in SoA
 * form.  Any per-problem pointer may be NULL to skip that field. */
typedef struct tb_batch_result {
    double* x_star;          /* [count][dim] */
    double* f_star;          /* [count] */
    double* pg_norm;         /* [count] */
    int32_t* status;         /* [count] TB_STATUS_* */
    int32_t* iterations;     /* [count] */
    int64_t* cg_iterations;  /* [count] (long in the reference) */
    int64_t* f_evals;        /* [count] */
    double* wall_time;       /* [count] seconds, per-problem device time (per_problem_time) */
    int64_t* flops;          /* [count] algorithmic FP64 flops (DESIGN.md model), optional */
    int32_t memspace;        /* where the per-problem arrays live */
    /* host-side aggregates, always written */
    double partition_times[64]; /* seconds per device partition (batch.hpp:20) */
    int32_t n_partitions;
    double batch_wall_time; /* seconds (batch.hpp:21) */
    double kernel_time;     /* seconds, max over devices of the solve kernel */
} tb_batch_result;

typedef struct tb_context tb_context;

/* TronConfig{} defaults (tron.hpp:55-68). */
void tb_config_default(tb_tron_config* cfg);
/* TronConfig::validate (tron.hpp:70-80): TB_OK or TB_E_INVALID_ARGUMENT with
 * the reference's message in tb_last_error(). */
int tb_config_validate(const tb_tron_config* cfg);

/* Parameters per problem for (family, dim); -1 if the pair is invalid. */
int64_t tb_family_nparams(int32_t family, int32_t dim);

/* Device context: one CUDA stream + reusable workspace per device.  The
 * reference's `workers` argument (batch.hpp:29) becomes the device list: the
 * batch is split in contiguous even partitions in input order over devices
 * (batch.hpp:61-70).  A context (its staging buffers, workspaces and host
 * thread team) serves one host thread at a time; use one context per host
 * thread that solves concurrently. */
int tb_context_create(const int32_t* devices, int32_t n_devices, tb_context** out);
int tb_context_destroy(tb_context* ctx);
/* mode must be TB_MODE_EXACT.  fast_forward: 1 (default) skips the provably
 * identical replays of a rejected zero-change iteration and
 * credits their flops to the per-problem flop counter (the reference's
 * count); 2 skips them and counts only the flops executed (also leaving out
 * the attempts of a memoised factorization); 0 replays them.
 * Every SolveReport field is identical in all three. */
int tb_context_set_mode(tb_context* ctx, int32_t mode, int32_t fast_forward);
/* Kernel form (TB_FORM_*, default TB_FORM_AUTO) for the context's later
 * solves; replaces the round-1 TB_THREAD / TB_BLOCK_* environment switches. */
int tb_context_set_form(tb_context* ctx, int32_t form);
/* Launch order (TB_ORDER_*, default TB_ORDER_AUTO) for the context's later
 * solves. */
int tb_context_set_order(tb_context* ctx, int32_t order);

/* solve_batch (batch.hpp:27-78): blocking.  Returns TB_E_PROBLEM if any
 * problem reports a status >= TB_STATUS_EVALUATION_ERROR (the reference would
 * have thrown); results are still written.  Dimensions 1..128: one warp per
 * problem up to d = 16, a block of 32 / 64 / 128 threads per problem above
 * (persistent grid, workspace owned by the context); larger d is rejected with
 * TB_E_INVALID_ARGUMENT. */
int tb_solve_batch(tb_context* ctx, const tb_problem_batch* batch, const tb_tron_config* cfg,
                   tb_batch_result* result);
/* Stream-ordered variant for device-resident batches on a single-device
 * context: enqueue on `stream` (a cudaStream_t, NULL = the context stream)
 * and return without synchronising.  Aggregates are not filled. */
int tb_solve_batch_async(tb_context* ctx, const tb_problem_batch* batch, const tb_tron_config* cfg,
                         tb_batch_result* result, void* stream);

/* Per-chunk host callbacks of tb_solve_batch_packed.  `pack` writes problems
 * [begin, end) into page-locked staging: x0 / lower / upper as
 * [end - begin][dim], params as [end - begin][nparams] (NULL when the family
 * has none).  `unpack` receives the results of problems [begin, end) as a host
 * tb_batch_result whose arrays start at problem `begin` (flops NULL); the
 * arrays are valid only during the call. */
typedef void (*tb_pack_fn)(void* user, int64_t begin, int64_t end, double* x0, double* lower, double* upper,
                           double* params);
typedef void (*tb_unpack_fn)(void* user, int64_t begin, int64_t end, const tb_batch_result* results);
/* solve_batch (batch.hpp:27-78) for callers whose problems are not laid out
 * as arrays (the C++ drop-in's std::vector<P>): the library asks for each
 * pipeline chunk's inputs just before copying them to the device and hands
 * over each chunk's results as soon as they arrive, so the caller's packing
 * and report building overlap the device work on the other chunks.  Errors
 * as tb_solve_batch; `result` receives the aggregates only.  The callbacks
 * run on the calling thread, in problem order. */
int tb_solve_batch_packed(tb_context* ctx, int32_t family, int32_t dim, int64_t count, const tb_tron_config* cfg,
                          tb_pack_fn pack, tb_unpack_fn unpack, void* user, tb_batch_result* result);

/* imbalance (batch.hpp:89-111): times is [n_iters][n_parts] row-major. */
int tb_imbalance(const double* times, int32_t n_iters, int32_t n_parts, double* nu_per_iter,
                 double* nu_max, double* nu_min, double* nu_mean);

const char* tb_last_error(void);
/* Number of kernels this library launched since load (TRON, block, error
 * scan and ADMM stage kernels; evidence counter for the bench). */
int64_t tb_kernel_launch_count(void);

/* Page-locked host memory (cudaHostAlloc, portable) for callers that pack
 * batches themselves (the C++ drop-in): tb_solve_batch copies page-locked
 * buffers straight into its chunked pipeline, without staging. */
int tb_host_alloc(int64_t bytes, void** out);
int tb_host_free(void* p);

/* FP64 DFMA throughput of `device` in TFLOP/s (the roofline denominator of
 * the TRON kernel; measured, not nominal). */
int tb_measure_fp64_peak(int32_t device, double* tflops);


/* ---- ADMM AC-OPF (the reference ships no code for it) ---
 * Device-resident component ADMM whose branch stage is the batched TRON
 * kernel.  One process per GPU: branches are sharded in equal chunks; after
 * tb_admm_solve_components the caller all-gathers the branch solutions (NCCL)
 * into the buffer of tb_admm_branch_solution, then tb_admm_update_consensus
 * runs the bus / multiplier / residual step and leaves this shard's residual
 * maxima (and branch-failure flag) for a max-allreduce.  Single process:
 * tb_admm_step, or tb_admm_run for a whole solve without per-iteration host
 * round trips. */
typedef struct tb_admm_grid {
    int32_t n_bus, n_gen, n_branch;
    const double *bus_pd, *bus_qd, *bus_gsh, *bus_bsh, *bus_vmin, *bus_vmax; /* [n_bus], per unit */
    const int32_t* gen_bus;                                                  /* [n_gen] */
    const double *gen_c2, *gen_c1, *gen_pmin, *gen_pmax, *gen_qmin, *gen_qmax;
    const int32_t *br_from, *br_to; /* [n_branch] */
    const double* br_coef;          /* [n_branch][8] pi-model flow coefficients (TB_BR_GFF..TB_BR_BTF) */
    const double* br_smax2;         /* [n_branch] line limit s-bar^2 (per unit^2, Eq. (2c)); read only with
                                       options.line_limits; NULL = unlimited */
} tb_admm_grid;

typedef struct tb_admm_options {
    double rho_pq; /* power couplings (rho0 = 10) */
    double rho_va; /* voltage / angle couplings (4 rho0) */
    int32_t shard_rank, shard_count;
    tb_tron_config tron;
    /* Line limits (SPEC.md:425 leaves Eq. (2c) out of
     * Eq. (3)): 0 = the SPEC's d = 4 branch subproblem; 1 = the d = 6 variant
     * with slacks s in [-s-bar^2, 0], h = p^2 + q^2 + s = 0 per line end,
     * enforced by an augmented-Lagrangian loop around the branch TRON solves
     * inside every ADMM iteration: solve the active branches, then per branch
     * with hmax = max |h|: hmax <= feas_tol -> done; hmax <= eta -> mu += xi h,
     * eta = max(feas_tol, 0.1 eta); else xi = min(xi_max, 10 xi).  mu carries
     * over between ADMM iterations, xi and eta restart at xi0 / eta0. */
    int32_t line_limits;
    int32_t auglag_max_iter; /* AL rounds per ADMM iteration (default 20) */
    double auglag_xi0;       /* default 10 */
    double auglag_xi_max;    /* default 1e8 */
    double auglag_eta0;      /* default 0.1 */
    double auglag_feas_tol;  /* default 1e-6 */
    /* d = 4 branch stage: TB_FORM_AUTO (one thread per branch, launched
     * together with the generator updates) or TB_FORM_WARP (one warp per
     * branch); results are identical */
    int32_t branch_form;
} tb_admm_options;

typedef struct tb_admm tb_admm;

#define TB_ADMM_GEN_P 0
#define TB_ADMM_GEN_Q 1
#define TB_ADMM_GEN_PT 2
#define TB_ADMM_GEN_QT 3
#define TB_ADMM_GEN_LP 4
#define TB_ADMM_GEN_LQ 5
#define TB_ADMM_BUS_WT 6
#define TB_ADMM_BUS_TT 7
#define TB_ADMM_BRANCH_X 8      /* [n_branch][dim] (v_i, v_j, th_i, th_j[, s_ij, s_ji]); dim 6 with line_limits */
#define TB_ADMM_BRANCH_PARAMS 9 /* [n_branch][36] incl. lambda / rho / consensus */
#define TB_ADMM_BRANCH_STATUS 10
#define TB_ADMM_COST 11 /* sum_g c2 p^2 + c1 p */
#define TB_ADMM_AUGLAG_ROUNDS 12 /* int64 [1]: AL rounds run so far (line_limits) */
#define TB_ADMM_LINE_VIOL 13     /* double [1]: max over branches and ends of |h| (line_limits) */
#define TB_ADMM_STAGE_TIMES 14   /* double [2]: seconds of the latest iteration's components (generators +
                                    branch TRON) and consensus stages, device events (per-partition batch
                                    time of SPEC.md:408) */

void tb_admm_options_default(tb_admm_options* opt);
/* x_external: optional device buffer for the branch solutions,
 * ceil(n_branch / shard_count) * shard_count rows of 4 doubles (NULL: owned) */
int tb_admm_create(const tb_admm_grid* grid, const tb_admm_options* opt, int32_t device, double* x_external,
                   tb_admm** out);
int tb_admm_destroy(tb_admm* a);
int tb_admm_solve_components(tb_admm* a, void* stream);
int tb_admm_branch_solution(tb_admm* a, double** x_dev, int64_t* lo, int64_t* hi);
/* res3_dev (device, 3 doubles, may be NULL): this shard's residual maxima and
 * its first failed branch (-1 none) -- max-allreduce them across shards. */
int tb_admm_update_consensus(tb_admm* a, void* stream, double* res3_dev);
/* One iteration, blocking: residuals to host.  TB_E_PROBLEM when a branch
 * solve ended where the reference throws ("propagated solver
 * failures"); the message names the branch and status. */
int tb_admm_step(tb_admm* a, double* primal, double* dual);
/* admm_solve, single shard: up to max_iter iterations, stop
 * at the first whose residuals are both <= tol; one captured CUDA graph per
 * iteration, a device stop flag, the host polls every check_every
 * iterations (no per-iteration round trip).  hist_out [max_iter][2] (NULL
 * allowed), *iters_out = iterations run.  TB_E_PROBLEM as tb_admm_step. */
int tb_admm_run(tb_admm* a, int32_t max_iter, double tol_primal, double tol_dual, int32_t check_every,
                double* hist_out, int32_t* iters_out);
/* Sharded path: first failed branch (global index, -1 none) since the last
 * call and its status; blocking; clears the record. */
int tb_admm_branch_errors(tb_admm* a, int64_t* first_bad, int32_t* status);
int tb_admm_get(tb_admm* a, int32_t what, void* host_out);
const char* tb_admm_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* TB_CAPI_H */
