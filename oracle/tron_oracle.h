/*
 * tron_oracle.h — TEST INFRASTRUCTURE ONLY.  CPU restatement (plain C99) of
 * the reference TRON path (/root/reference/proj/include/tronbatch/{dense,
 * tron,batch}.hpp).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it, and only as the checker.  The product path
 * (paper_2106_14995_b200/) never links it.
 *
 * Pinned against (a) the reference's own unit tests, compiled unmodified
 * against oracle/compat/ (C++ adapter over this file) and (b) bitwise equality
 * with the reference headers compiled into oracle/_ref/libtronref.so.
 */
#ifndef TRON_ORACLE_H
#define TRON_ORACLE_H

#include <stdint.h>

#include "../include/tb_capi.h"

#ifdef __cplusplus
extern "C" {
#endif

/* BoundedProblem (tron.hpp:28-36) as a C callback bundle. */
typedef struct orc_problem {
    int n;
    const double* lower;
    const double* upper;
    double (*f)(void* ctx, const double* x);
    void (*grad)(void* ctx, const double* x, double* g);
    void (*hess)(void* ctx, const double* x, double* A); /* col-major n x n */
    void* ctx;
} orc_problem;

/* SolveReport (tron.hpp:94-103) minus x_star/wall_time (written separately). */
typedef struct orc_report {
    double f_star;
    double pg_norm;
    int32_t status;
    int32_t iterations;
    int64_t cg_iterations;
    int64_t f_evals;
    int64_t flops; /* algorithmic flop model */
    int32_t executed_iterations; /* loop iterations actually run */
    int32_t ff_iter;             /* first zero-change fixed-point iteration, 0 if none */
} orc_report;

/* Opt-in fast-forward of zero-change fixed points (as the device does). */
void orc_set_fast_forward(int on);

/* dense.hpp */
void orc_axpy(int n, double alpha, const double* x, double* y);
double orc_dot(int n, const double* x, const double* y);
double orc_nrm2(int n, const double* x);
void orc_scal(int n, double alpha, double* x);
void orc_gemv(int n, double alpha, const double* A, const double* x, double beta, double* y,
              int transpose);
void orc_ccfs(int n, double* A, double alpha);
int orc_chol_left(int n, const double* A, double shift, double* L);
int orc_chol_right(int n, const double* A, double shift, double* L);
/* returns 0, or TB_STATUS_FACTORIZATION_FAILED */
int orc_ccf(int n, const double* A, double* L, double* shift);
int orc_ccf_right(int n, const double* A, double* L, double* shift);
/* returns 0, or TB_STATUS_SINGULAR_FACTOR */
int orc_trtrs(int n, const double* L, double* b, int transpose);
double orc_max_abs(int n, const double* A);

/* tron.hpp */
void orc_clip(int n, double* x, const double* l, const double* u);
double orc_pgnorm(int n, const double* x, const double* g, const double* l, const double* u);
void orc_gpstep(int n, const double* x, double alpha, const double* w, const double* l,
                const double* u, double* s);
void orc_breakpt(int n, const double* x, const double* w, const double* l, const double* u,
                 int* count, double* bmin, double* bmax);
/* returns 0 or TB_STATUS_ZERO_DIRECTION */
int orc_trqsol(int n, const double* x, const double* w, double delta, double* sigma);
double orc_quad_model(int n, const double* A, const double* g, const double* s);
/* returns 0 or TB_STATUS_EVALUATION_ERROR */
int orc_cauchy(int n, const double* x, const double* g, const double* A, const double* l,
               const double* u, double delta, const tb_tron_config* cfg, double alpha_start,
               double* alpha_out, double* s);
int orc_select_free_set(int n, const double* x, const double* l, const double* u, int* free_set);
/* CgStatus: 0 Converged, 1 Boundary, 2 NegCurve, 3 IterCap; returns 0 or error */
int orc_precond_cg(int n, const double* A, const double* g, const double* L, double delta,
                   const tb_tron_config* cfg, double* step, int* cg_status, int* iterations,
                   double* rel_residual);
void orc_line_search(int n, const double* x, const double* l, const double* u, const double* A,
                     const double* g, const double* w, const tb_tron_config* cfg, double* beta,
                     double* x_next);
/* solve(): returns 0 or a status >= TB_STATUS_EVALUATION_ERROR (the
 * reference would throw); rep is always filled. */
int orc_solve(const orc_problem* p, const double* x0, const tb_tron_config* cfg, double* x_star,
              orc_report* rep);

/* family twins (csrc/tb_families.h) */
int orc_solve_family(int family, int n, const double* x0, const double* l, const double* u,
                     const double* params, const tb_tron_config* cfg, double* x_star,
                     orc_report* rep);
/* solve_batch (batch.hpp:27-78) over `workers` pthreads, static even
 * partition.  Returns 0 or the first (in partition order) error status. */
int orc_solve_batch(int family, int n, int64_t count, const double* x0, const double* lower,
                    const double* upper, const double* params, int64_t params_stride,
                    const tb_tron_config* cfg, int workers, double* x_star, double* f_star,
                    double* pg_norm, int32_t* status, int32_t* iterations, int64_t* cg_iterations,
                    int64_t* f_evals, int64_t* flops, int32_t* executed, int32_t* ff_iter,
                    double* batch_wall_time);
/* family f/grad/Hessian (for derivative tests) */
void orc_family_eval(int family, int n, const double* x, const double* params, double* f,
                     double* g, double* H);
int orc_imbalance(const double* times, int n_iters, int n_parts, double* nu, double* nu_max,
                  double* nu_min, double* nu_mean);
void orc_config_default(tb_tron_config* cfg);
/* returns 0 or 1 (invalid) with a message */
int orc_config_validate(const tb_tron_config* cfg, const char** msg);

#ifdef __cplusplus
}
#endif

#endif
