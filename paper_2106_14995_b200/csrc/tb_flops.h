/*
 * tb_flops.h — the algorithmic FP64 flop model,
 * shared by the device kernel's per-problem counters and the CPU oracle so
 * that both report the same number for the same executed path.
 *
 * Counted as executed (n = the operation's active dimension; FMA = 2):
 *   dot 2n   nrm2 2n+1   axpy 2n   scal n   gpstep 2n   breakpt 2n
 *   gemv 2n per non-skipped column (dense.hpp:110 zero-skip)
 *   trtrs n^2            quad_model = gemv + 2 dots + 2
 *   trqsol 3 dots + 8    cholesky column j of an nf-system: 2(nf-j) per
 *   non-skipped k (dense.hpp:146) + 2 + (nf-j-1)
 *   family f / grad / Hessian evaluations: tb_family_flops below.
 * Comparisons, clips and max-reductions are not counted.
 */
#ifndef TB_FLOPS_H
#define TB_FLOPS_H

#include "tb_math.h"

#define TB_FLOPS_SINCOS 25

/* kind: 0 = f, 1 = full gradient, 2 = full Hessian */
TB_HD long long tb_family_flops(int fam, int n, int kind) {
    const long long N = n;
    switch (fam) {
        case 0: /* hs45 */
            return kind == 0 ? N + 1 : (kind == 1 ? 3 * N : N * N);
        case 1: /* boxqp */
            return kind == 0 ? 2 * N * N + 3 * N + 1 : (kind == 1 ? 2 * N * N + N : 0);
        case 2: /* ncvx */
            return kind == 0 ? 2 * N * N + (10 + TB_FLOPS_SINCOS) * N + 3
                             : (kind == 1 ? 2 * N * N + (6 + TB_FLOPS_SINCOS) * N
                                          : (5 + TB_FLOPS_SINCOS) * N);
        default: { /* branch, dim 4 or 6 */
            const long long ctx = TB_FLOPS_SINCOS + 117 + (n == 6 ? 44 : 0);
            if (kind == 0) return ctx + (n == 6 ? 50 : 40);
            if (kind == 1) return ctx + 10 * N + (n == 6 ? 16 : 0);
            return ctx + N * N * (40 + (n == 6 ? 38 : 0));
        }
    }
}

#endif /* TB_FLOPS_H */
