/*
 * tb_math.h — portable, bit-reproducible FP64 helpers shared by the device
 * kernels and the host problem twins used by the CPU oracle.
 *
 * Every function here is plain IEEE-754 double arithmetic (+, -, *, /, sqrt,
 * floor) written in a fixed evaluation order.  Compiled with gcc
 * `-ffp-contract=off` on x86-64 (SSE2, no FMA) and with nvcc `--fmad=false`
 * on sm_100a, the host and device produce identical bits.  CUDA's libm
 * sin/cos are NOT glibc's, so the problem families never call them.
 *
 * std::min / std::max semantics of libstdc++ (used throughout the reference,
 * e.g. tron.hpp:106,118,173,478) are reproduced exactly by tb_smin/tb_smax:
 *   std::max(a,b) == (a < b) ? b : a      std::min(a,b) == (b < a) ? b : a
 * which differ from fmax/fmin on NaN and on signed zeros.
 */
#ifndef TB_MATH_H
#define TB_MATH_H

#include <math.h>

#if defined(__CUDACC__)
#define TB_HD static inline __host__ __device__
#else
#define TB_HD static inline
#endif

TB_HD double tb_smax(double a, double b) { return (a < b) ? b : a; }
TB_HD double tb_smin(double a, double b) { return (b < a) ? b : a; }

/* 2^t for 0 <= t <= 1023, exact */
TB_HD double tb_pow2(int t) {
    union {
        unsigned long long u;
        double d;
    } v;
    v.u = (unsigned long long)(1023 + t) << 52;
    return v.d;
}

/* t steps of the shift escalation a <- std::max(2 a, alpha0) (dense.hpp:197)
 * at once, for a >= 0 and alpha0 > 0 (0 <= t <= 1000): doubling is exact
 * and std::max returns one of its operands, so by induction the t-th iterate
 * is max(2^t a, 2^(t-1) alpha0) bit for bit (an overflow gives inf both
 * ways).  Takes the shift of a parallel attempt group off a serial chain. */
TB_HD double tb_shift_ahead(double a, double alpha0, int t) {
    const double s = tb_smax(a * tb_pow2(t), alpha0 * tb_pow2(t > 0 ? t - 1 : 0));
    return t > 0 ? s : a;  // a select: t differs between the lane groups of a warp
}

/* fdlibm-style Cody-Waite reduction by pi/2 (33-bit head + tail) and the
 * fdlibm minimax kernels on [-pi/4, pi/4].  Accurate to ~1 ulp for |x| < 1e5,
 * deterministic everywhere; returns NaN for non-finite input. */
#define TB_INVPIO2 6.36619772367581382433e-01
#define TB_PIO2_1 1.57079632673412561417e+00
#define TB_PIO2_1T 6.07710050650619224932e-11

TB_HD double tb_kernel_sin(double x) {
    const double S1 = -1.66666666666666324348e-01, S2 = 8.33333333332248946124e-03,
                 S3 = -1.98412698298579493134e-04, S4 = 2.75573137070700676789e-06,
                 S5 = -2.50507602534068634195e-08, S6 = 1.58969099521155010221e-10;
    const double z = x * x;
    const double v = z * x;
    const double r = S2 + z * (S3 + z * (S4 + z * (S5 + z * S6)));
    return x + v * (S1 + z * r);
}

TB_HD double tb_kernel_cos(double x) {
    const double C1 = 4.16666666666666019037e-02, C2 = -1.38888888888741095749e-03,
                 C3 = 2.48015872894767294178e-05, C4 = -2.75573143513906633035e-07,
                 C5 = 2.08757232129817482790e-09, C6 = -1.13596475577881948265e-11;
    const double z = x * x;
    const double r = z * (C1 + z * (C2 + z * (C3 + z * (C4 + z * (C5 + z * C6)))));
    const double hz = 0.5 * z;
    const double w = 1.0 - hz;
    return w + (((1.0 - w) - hz) + z * r);
}

TB_HD void tb_sincos(double x, double* s, double* c) {
    if (!(x - x == 0.0)) { /* inf or NaN */
        *s = x - x;
        *c = x - x;
        return;
    }
    const double fn = floor(x * TB_INVPIO2 + 0.5);
    const double y = (x - fn * TB_PIO2_1) - fn * TB_PIO2_1T;
    const double ks = tb_kernel_sin(y);
    const double kc = tb_kernel_cos(y);
    const long long q = ((long long)fn) & 3LL;
    if (q == 0) { *s = ks;  *c = kc; }
    else if (q == 1) { *s = kc;  *c = -ks; }
    else if (q == 2) { *s = -ks; *c = -kc; }
    else { *s = -kc; *c = ks; }
}

TB_HD double tb_sin(double x) { double s, c; tb_sincos(x, &s, &c); return s; }
TB_HD double tb_cos(double x) { double s, c; tb_sincos(x, &s, &c); return c; }

#endif /* TB_MATH_H */
