/*
 * tb_admm_host.h — host-side ADMM set-up shared by the device path
 * (admm.cu, tb_admm_create) and the CPU oracle (oracle/admm_oracle.c):
 * incidence CSR in canonical order and the initial state (SPEC.md:426-427:
 * rho0 for power couplings, 4 rho0 for voltage couplings, flat start
 * v = 1, th = 0, lambda = 0; initial consensus = the component values at the
 * flat start / generator box midpoints).
 */
#ifndef TB_ADMM_HOST_H
#define TB_ADMM_HOST_H

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/tb_capi.h"
#include "tb_admm.h"

typedef struct {
    double *bus_wt, *bus_tt;
    double *gen_p, *gen_q, *gen_lp, *gen_lq, *gen_rp, *gen_rq, *gen_pt, *gen_qt;
    double *br_params, *br_x, *br_lower, *br_upper;
    int32_t *gen_ptr, *gen_idx, *end_ptr, *end_idx;
    int dim; /* branch dimension: 4, or 6 with line limits */
    char err[256];
} tb_admm_host_state;

static inline void tb_admm_host_free(tb_admm_host_state* s) {
    void* ps[] = {s->bus_wt, s->bus_tt, s->gen_p, s->gen_q, s->gen_lp, s->gen_lq, s->gen_rp, s->gen_rq,
                  s->gen_pt, s->gen_qt, s->br_params, s->br_x, s->br_lower, s->br_upper, s->gen_ptr,
                  s->gen_idx, s->end_ptr, s->end_idx};
    for (size_t k = 0; k < sizeof ps / sizeof ps[0]; ++k) free(ps[k]);
    memset(s, 0, sizeof(*s));
}

static inline int tb_admm_host_init(const tb_admm_grid* g, const tb_admm_options* o, tb_admm_host_state* s) {
    const int nb = g->n_bus, ng = g->n_gen, nl = g->n_branch;
    const double two_pi = 2.0 * 3.14159265358979323846;
    memset(s, 0, sizeof(*s));
    const int D = o->line_limits ? 6 : 4;
    s->dim = D;
#define TB_A(p, T, n) (p) = (T*)calloc((size_t)((n) > 0 ? (n) : 1), sizeof(T))
    TB_A(s->bus_wt, double, nb);
    TB_A(s->bus_tt, double, nb);
    TB_A(s->gen_p, double, ng);
    TB_A(s->gen_q, double, ng);
    TB_A(s->gen_lp, double, ng);
    TB_A(s->gen_lq, double, ng);
    TB_A(s->gen_rp, double, ng);
    TB_A(s->gen_rq, double, ng);
    TB_A(s->gen_pt, double, ng);
    TB_A(s->gen_qt, double, ng);
    TB_A(s->br_params, double, (long)nl * TB_BR_NPARAMS);
    TB_A(s->br_x, double, (long)nl * D);
    TB_A(s->br_lower, double, (long)nl * D);
    TB_A(s->br_upper, double, (long)nl * D);
    TB_A(s->gen_ptr, int32_t, nb + 1);
    TB_A(s->gen_idx, int32_t, ng);
    TB_A(s->end_ptr, int32_t, nb + 1);
    TB_A(s->end_idx, int32_t, 2 * nl);
#undef TB_A
    /* incidence CSR: counting sort, canonical order */
    for (int k = 0; k < ng; ++k) s->gen_ptr[g->gen_bus[k] + 1]++;
    for (int b = 0; b < nb; ++b) s->gen_ptr[b + 1] += s->gen_ptr[b];
    {
        int32_t* fill = (int32_t*)calloc((size_t)nb + 1, sizeof(int32_t));
        memcpy(fill, s->gen_ptr, sizeof(int32_t) * (size_t)(nb + 1));
        for (int k = 0; k < ng; ++k) s->gen_idx[fill[g->gen_bus[k]]++] = k;
        for (int l = 0; l < nl; ++l) {
            s->end_ptr[g->br_from[l] + 1]++;
            s->end_ptr[g->br_to[l] + 1]++;
        }
        for (int b = 0; b < nb; ++b) s->end_ptr[b + 1] += s->end_ptr[b];
        memcpy(fill, s->end_ptr, sizeof(int32_t) * (size_t)(nb + 1));
        for (int l = 0; l < nl; ++l) {
            s->end_idx[fill[g->br_from[l]]++] = 2 * l;
            s->end_idx[fill[g->br_to[l]]++] = 2 * l + 1;
        }
        free(fill);
    }
    for (int b = 0; b < nb; ++b) {
        s->bus_wt[b] = 1.0;
        s->bus_tt[b] = 0.0;
    }
    for (int k = 0; k < ng; ++k) {
        s->gen_rp[k] = o->rho_pq;
        s->gen_rq[k] = o->rho_pq;
        s->gen_p[k] = s->gen_pt[k] = 0.5 * (g->gen_pmin[k] + g->gen_pmax[k]);
        s->gen_q[k] = s->gen_qt[k] = 0.5 * (g->gen_qmin[k] + g->gen_qmax[k]);
    }
    for (int l = 0; l < nl; ++l) {
        double* prm = s->br_params + (long)l * TB_BR_NPARAMS;
        double* x = s->br_x + (long)l * D;
        for (int k = 0; k < 8; ++k) prm[k] = g->br_coef[(long)l * 8 + k];
        x[0] = 1.0;
        x[1] = 1.0;
        x[2] = 0.0;
        x[3] = 0.0;
        double base[8];
        tb_br_base(x, base);
        for (int f = 0; f < 4; ++f) {
            prm[TB_BR_LAM + f] = 0.0;
            prm[TB_BR_RHO + f] = o->rho_pq;
            prm[TB_BR_TIL + f] = tb_admm_flow(base, prm, f);
        }
        for (int e = 0; e < 2; ++e) {
            prm[TB_BR_LAMW + e] = 0.0;
            prm[TB_BR_RHOW + e] = o->rho_va;
            prm[TB_BR_WTIL + e] = 1.0;
            prm[TB_BR_LAMT + e] = 0.0;
            prm[TB_BR_RHOT + e] = o->rho_va;
            prm[TB_BR_TTIL + e] = 0.0;
        }
        const int fb = g->br_from[l], tb = g->br_to[l];
        double* lo = s->br_lower + (long)l * D;
        double* up = s->br_upper + (long)l * D;
        lo[0] = g->bus_vmin[fb];
        lo[1] = g->bus_vmin[tb];
        lo[2] = -two_pi;
        lo[3] = -two_pi;
        up[0] = g->bus_vmax[fb];
        up[1] = g->bus_vmax[tb];
        up[2] = two_pi;
        up[3] = two_pi;
        if (D == 6) { /* slacks s in [-s-bar^2, 0], started at the flat-start flows */
            const double sm2 = g->br_smax2 ? g->br_smax2[l] : HUGE_VAL;
            if (!(sm2 >= 0.0)) {
                snprintf(s->err, sizeof s->err, "tb_admm_create: branch %d line limit s-bar^2 must be >= 0", l);
                return 1;
            }
            prm[TB_BR_MU] = prm[TB_BR_MU + 1] = 0.0;
            prm[TB_BR_XI] = o->auglag_xi0;
            prm[TB_BR_SMAX2] = sm2;
            for (int e = 0; e < 2; ++e) {
                const double p = tb_admm_flow(base, prm, 2 * e), q = tb_admm_flow(base, prm, 2 * e + 1);
                lo[4 + e] = -sm2;
                up[4 + e] = 0.0;
                x[4 + e] = tb_smax(-(p * p + q * q), -sm2);
            }
        }
    }
    return 0;
}

#endif /* TB_ADMM_HOST_H */
