/*
 * admm_oracle.c — TEST INFRASTRUCTURE ONLY.  CPU restatement of the
 * component ADMM of SPEC.md:319-441 (the reference has no code for it):
 * generator closed form, branch subproblems through the C TRON restatement
 * (orc_solve_batch, bit-identical to the reference solve_batch), bus
 * consensus / multipliers / residuals — the closed forms are the shared
 * plain-C functions of csrc/tb_admm.h, evaluated sequentially in canonical
 * order.  Parity with the device is therefore exact (same bits per iteration);
 * the spec's own examples pin the closed forms (tests/test_admm.py).  With
 * line limits (options.line_limits) the branch stage is the augmented-
 * Lagrangian loop of tb_admm_options, restated here in ascending order.
 */
#include <stdlib.h>
#include <string.h>

#include "../paper_2106_14995_b200/csrc/tb_admm_host.h"
#include "tron_oracle.h"

typedef struct orc_admm {
    tb_admm_host_state hs;
    tb_admm_view v;
    tb_admm_options opt;
    int workers;
    int nb, ng, nl;
    double *pd, *qd, *gsh, *bsh, *c2, *c1, *pmin, *pmax, *qmin, *qmax, *xtmp;
    int32_t *gen_bus, *from, *to, *status;
    int dim;                                /* 4, or 6 with line limits */
    double *eta, *cx, *cl, *cu, *cp, *cxo;  /* augmented-Lagrangian state / compaction */
    int32_t *active, *cidx, *cst;
    long auglag_rounds;
} orc_admm;

static double* dup_d(const double* s, int n) {
    double* d = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    if (n > 0) memcpy(d, s, sizeof(double) * (size_t)n);
    return d;
}
static int32_t* dup_i(const int32_t* s, int n) {
    int32_t* d = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    if (n > 0) memcpy(d, s, sizeof(int32_t) * (size_t)n);
    return d;
}

int orc_admm_create(const tb_admm_grid* g, const tb_admm_options* o, int workers, orc_admm** out) {
    orc_admm* a = (orc_admm*)calloc(1, sizeof(orc_admm));
    a->opt = *o;
    a->workers = workers < 1 ? 1 : workers;
    a->nb = g->n_bus;
    a->ng = g->n_gen;
    a->nl = g->n_branch;
    if (tb_admm_host_init(g, o, &a->hs) != 0) {
        free(a);
        return 1;
    }
    a->pd = dup_d(g->bus_pd, a->nb);
    a->qd = dup_d(g->bus_qd, a->nb);
    a->gsh = dup_d(g->bus_gsh, a->nb);
    a->bsh = dup_d(g->bus_bsh, a->nb);
    a->c2 = dup_d(g->gen_c2, a->ng);
    a->c1 = dup_d(g->gen_c1, a->ng);
    a->pmin = dup_d(g->gen_pmin, a->ng);
    a->pmax = dup_d(g->gen_pmax, a->ng);
    a->qmin = dup_d(g->gen_qmin, a->ng);
    a->qmax = dup_d(g->gen_qmax, a->ng);
    a->gen_bus = dup_i(g->gen_bus, a->ng);
    a->from = dup_i(g->br_from, a->nl);
    a->to = dup_i(g->br_to, a->nl);
    a->dim = a->hs.dim;
    a->xtmp = (double*)malloc(sizeof(double) * a->dim * (size_t)a->nl);
    a->status = (int32_t*)malloc(sizeof(int32_t) * (size_t)a->nl);
    if (a->dim == 6) {
        const size_t m = (size_t)(a->nl > 0 ? a->nl : 1);
        a->eta = (double*)malloc(sizeof(double) * m);
        a->cx = (double*)malloc(sizeof(double) * 6 * m);
        a->cl = (double*)malloc(sizeof(double) * 6 * m);
        a->cu = (double*)malloc(sizeof(double) * 6 * m);
        a->cxo = (double*)malloc(sizeof(double) * 6 * m);
        a->cp = (double*)malloc(sizeof(double) * TB_BR_NPARAMS * m);
        a->active = (int32_t*)malloc(sizeof(int32_t) * m);
        a->cidx = (int32_t*)malloc(sizeof(int32_t) * m);
        a->cst = (int32_t*)malloc(sizeof(int32_t) * m);
    }
    tb_admm_view* v = &a->v;
    v->n_bus = a->nb;
    v->n_gen = a->ng;
    v->n_branch = a->nl;
    v->branch_dim = a->dim;
    v->bus_pd = a->pd;
    v->bus_qd = a->qd;
    v->bus_gsh = a->gsh;
    v->bus_bsh = a->bsh;
    v->bus_wt = a->hs.bus_wt;
    v->bus_tt = a->hs.bus_tt;
    v->gen_bus = a->gen_bus;
    v->gen_c2 = a->c2;
    v->gen_c1 = a->c1;
    v->gen_pmin = a->pmin;
    v->gen_pmax = a->pmax;
    v->gen_qmin = a->qmin;
    v->gen_qmax = a->qmax;
    v->gen_p = a->hs.gen_p;
    v->gen_q = a->hs.gen_q;
    v->gen_lp = a->hs.gen_lp;
    v->gen_lq = a->hs.gen_lq;
    v->gen_rp = a->hs.gen_rp;
    v->gen_rq = a->hs.gen_rq;
    v->gen_pt = a->hs.gen_pt;
    v->gen_qt = a->hs.gen_qt;
    v->br_from = a->from;
    v->br_to = a->to;
    v->br_params = a->hs.br_params;
    v->br_x = a->hs.br_x;
    v->gen_ptr = a->hs.gen_ptr;
    v->gen_idx = a->hs.gen_idx;
    v->end_ptr = a->hs.end_ptr;
    v->end_idx = a->hs.end_idx;
    *out = a;
    return 0;
}

/* Branch stage for rows [lo, hi): one warm-started batched TRON solve (d = 4),
 * or the augmented-Lagrangian rounds of the line-limit variant (d = 6, see
 * tb_admm_options in include/tb_capi.h): solve the active branches (compacted
 * in ascending order), then tb_admm_auglag_update per solved branch. */
static int orc_branch_stage(orc_admm* a, int64_t lo, int64_t hi) {
    const int D = a->dim;
    if (hi <= lo) return 0;
    const int64_t cnt = hi - lo;
    if (D == 4) {
        const int rc = orc_solve_batch(TB_FAMILY_BRANCH, 4, cnt, a->hs.br_x + lo * 4, a->hs.br_lower + lo * 4,
                                       a->hs.br_upper + lo * 4, a->hs.br_params + lo * TB_BR_NPARAMS,
                                       TB_BR_NPARAMS, &a->opt.tron, a->workers, a->xtmp, NULL, NULL, a->status + lo,
                                       NULL, NULL, NULL, NULL, NULL, NULL, NULL);
        memcpy(a->hs.br_x + lo * 4, a->xtmp, sizeof(double) * 4 * (size_t)cnt);
        return rc;
    }
    for (int64_t l = lo; l < hi; ++l) {
        a->hs.br_params[l * TB_BR_NPARAMS + TB_BR_XI] = a->opt.auglag_xi0;
        a->eta[l] = a->opt.auglag_eta0;
        a->active[l] = 1;
    }
    int rc = 0;
    for (int round = 0; round < a->opt.auglag_max_iter; ++round) {
        int64_t m = 0;
        for (int64_t l = lo; l < hi; ++l) {
            if (!a->active[l]) continue;
            a->cidx[m] = (int32_t)l;
            memcpy(a->cx + m * 6, a->hs.br_x + l * 6, sizeof(double) * 6);
            memcpy(a->cl + m * 6, a->hs.br_lower + l * 6, sizeof(double) * 6);
            memcpy(a->cu + m * 6, a->hs.br_upper + l * 6, sizeof(double) * 6);
            memcpy(a->cp + m * TB_BR_NPARAMS, a->hs.br_params + l * TB_BR_NPARAMS, sizeof(double) * TB_BR_NPARAMS);
            ++m;
        }
        if (m == 0) break;
        ++a->auglag_rounds;
        const int r = orc_solve_batch(TB_FAMILY_BRANCH, 6, m, a->cx, a->cl, a->cu, a->cp, TB_BR_NPARAMS,
                                      &a->opt.tron, a->workers, a->cxo, NULL, NULL, a->cst, NULL, NULL, NULL, NULL,
                                      NULL, NULL, NULL);
        if (r && !rc) rc = r;
        for (int64_t k = 0; k < m; ++k) {
            const int64_t l = a->cidx[k];
            double* x = a->hs.br_x + l * 6;
            memcpy(x, a->cxo + k * 6, sizeof(double) * 6);
            a->status[l] = a->cst[k];
            a->active[l] = tb_admm_auglag_update(x, a->hs.br_params + l * TB_BR_NPARAMS, a->eta + l,
                                                 a->opt.auglag_feas_tol, a->opt.auglag_xi_max);
        }
    }
    return rc;
}

/* One iteration. Returns 0 or the TRON error status. */
int orc_admm_step(orc_admm* a, double* primal, double* dual) {
    for (int g = 0; g < a->ng; ++g) tb_admm_gen_update(&a->v, g);
    const int rc = orc_branch_stage(a, 0, a->nl);
    double pr = 0.0, du = 0.0;
    for (int b = 0; b < a->nb; ++b) {
        tb_admm_res r;
        tb_admm_bus_update(&a->v, b, &r);
        if (pr < r.primal) pr = r.primal;
        if (du < r.dual) du = r.dual;
    }
    *primal = pr;
    *dual = du;
    return rc;
}

int orc_admm_get(orc_admm* a, int what, void* out) {
    const void* src = NULL;
    size_t bytes = 0;
    switch (what) {
        case TB_ADMM_GEN_P: src = a->hs.gen_p; bytes = sizeof(double) * a->ng; break;
        case TB_ADMM_GEN_Q: src = a->hs.gen_q; bytes = sizeof(double) * a->ng; break;
        case TB_ADMM_GEN_PT: src = a->hs.gen_pt; bytes = sizeof(double) * a->ng; break;
        case TB_ADMM_GEN_QT: src = a->hs.gen_qt; bytes = sizeof(double) * a->ng; break;
        case TB_ADMM_GEN_LP: src = a->hs.gen_lp; bytes = sizeof(double) * a->ng; break;
        case TB_ADMM_GEN_LQ: src = a->hs.gen_lq; bytes = sizeof(double) * a->ng; break;
        case TB_ADMM_BUS_WT: src = a->hs.bus_wt; bytes = sizeof(double) * a->nb; break;
        case TB_ADMM_BUS_TT: src = a->hs.bus_tt; bytes = sizeof(double) * a->nb; break;
        case TB_ADMM_BRANCH_X: src = a->hs.br_x; bytes = sizeof(double) * a->dim * (size_t)a->nl; break;
        case TB_ADMM_AUGLAG_ROUNDS: *(int64_t*)out = a->auglag_rounds; return 0;
        case TB_ADMM_LINE_VIOL: {
            if (a->dim != 6) return 1;
            double m = 0.0, h[2];
            for (int l = 0; l < a->nl; ++l) {
                double v = tb_admm_line_hmax(a->hs.br_x + (long)l * 6, a->hs.br_params + (long)l * TB_BR_NPARAMS, h);
                if (!(v >= 0.0)) v = 1.0 / 0.0;
                if (m < v) m = v;
            }
            *(double*)out = m;
            return 0;
        }
        case TB_ADMM_BRANCH_PARAMS: src = a->hs.br_params; bytes = sizeof(double) * TB_BR_NPARAMS * (size_t)a->nl; break;
        case TB_ADMM_BRANCH_STATUS: src = a->status; bytes = sizeof(int32_t) * (size_t)a->nl; break;
        case TB_ADMM_COST: {
            double s = 0.0;
            for (int g = 0; g < a->ng; ++g) s += tb_admm_gen_cost(&a->v, g);
            *(double*)out = s;
            return 0;
        }
        default: return 1;
    }
    memcpy(out, src, bytes);
    return 0;
}

void orc_admm_destroy(orc_admm* a) {
    if (!a) return;
    tb_admm_host_free(&a->hs);
    void* ps[] = {a->pd, a->qd, a->gsh, a->bsh, a->c2, a->c1, a->pmin, a->pmax, a->qmin, a->qmax,
                  a->xtmp, a->gen_bus, a->from, a->to, a->status, a->eta, a->cx, a->cl, a->cu, a->cp, a->cxo,
                  a->active, a->cidx, a->cst};
    for (size_t k = 0; k < sizeof ps / sizeof ps[0]; ++k) free(ps[k]);
    free(a);
}

/* closed-form unit hooks for the SPEC examples */
double orc_admm_gen_p(double c2, double c1, double lam, double rho, double ptil, double pmin, double pmax) {
    double p = 0, q = 0, lq = 0, rq = 1, qt = 0, qmin = -1, qmax = 1;
    int32_t bus = 0;
    tb_admm_view v;
    memset(&v, 0, sizeof v);
    v.gen_c2 = &c2; v.gen_c1 = &c1; v.gen_lp = &lam; v.gen_rp = &rho; v.gen_pt = &ptil;
    v.gen_pmin = &pmin; v.gen_pmax = &pmax; v.gen_p = &p; v.gen_q = &q; v.gen_lq = &lq;
    v.gen_rq = &rq; v.gen_qt = &qt; v.gen_qmin = &qmin; v.gen_qmax = &qmax; v.gen_bus = &bus;
    tb_admm_gen_update(&v, 0);
    return p;
}

/* ---- phases (the sharded scheme of paper_2106_14995_b200/admm.py, on CPU) */
/* generator update (all) + branch TRON for rows [lo, hi) in place */
int orc_admm_solve_components(orc_admm* a, int64_t lo, int64_t hi) {
    for (int g = 0; g < a->ng; ++g) tb_admm_gen_update(&a->v, g);
    return orc_branch_stage(a, lo, hi);
}
double* orc_admm_x(orc_admm* a) { return a->hs.br_x; }
/* bus update over every bus; residual maxima over buses [blo, bhi) */
void orc_admm_update_consensus(orc_admm* a, int blo, int bhi, double* primal, double* dual) {
    double pr = 0.0, du = 0.0;
    for (int b = 0; b < a->nb; ++b) {
        tb_admm_res r;
        tb_admm_bus_update(&a->v, b, &r);
        if (b < blo || b >= bhi) continue;
        if (pr < r.primal) pr = r.primal;
        if (du < r.dual) du = r.dual;
    }
    *primal = pr;
    *dual = du;
}
