// glibc 2.39's x86-64 FMA builds of `log` and `sincos`, restated operation for operation
// so that the device Gaussian generator reproduces the reference's Omega bit for bit.
//
// Why: the reference draws Omega with std::log and a std::sin/std::cos pair on the same
// angle (rng.cpp:39-43), which gcc -O3 merges into one `sincos` call; on an AVX2+FMA host
// the glibc ifuncs resolve to __log_fma (sysdeps/ieee754/dbl-64/e_log.c, the
// table-driven ARM optimized-routines log) and __sincos_fma (s_sincos.c over s_sin.c's
// do_sin / do_cos / reduce_sincos, the IBM tables). Neither is correctly rounded, so a
// correctly rounded generator misses ~0.2 % of entries by an ulp. glibc is a third-party
// dependency the reference neither vendors nor pins; the pinned version here is this
// image's Ubuntu glibc 2.39-0ubuntu8.5.
//
// How: every arithmetic step below is one instruction of the compiled FMA builds (gcc
// contracted the C sources into fused multiply-adds; the contraction pattern is what
// decides the last bit, so it is restated from the machine code, `objdump -d libm.so.6`
// at __log_fma / __sincos_fma), with the glibc C expression each step implements in the
// comment. Every step is an explicit single rounding (rn_* helpers) so that neither nvcc
// nor the host compiler can re-contract it. The data (log tables, __sincostab, scalar
// constants) come from the same libm via tools/gen_glibc_tables.py.
//
// Domain: log for finite x > 0 in the normal range (the generator's uniforms are
// ((w >> 11) + 1) 2^-53 in [2^-53, 1]); sincos for |x| < 105414350 (the generator's
// angles are 2 pi u in (0, 2 pi]). The large-argument branch of sincos (branred) and
// log's subnormal/special inputs are outside the generator's domain and not restated.
// Checked against the host libm by tests/test_glibc_libm.py (host build of this header)
// and on the device by tests/test_gpu_parity.py (Omega == reference Omega, array_equal).
#pragma once

#include <stdint.h>
#include <string.h>

#include "glibc239_tables.h"

#if defined(__CUDACC__)
#define GLIBC_HD __host__ __device__ __forceinline__
#else
#define GLIBC_HD inline
#include <cmath>
#endif

namespace glibc239 {

#if defined(__CUDA_ARCH__)
__device__ const double kLogTab[256] = GLIBC239_LOG_TAB_INIT;
__device__ const double kSinCosTab[440] = GLIBC239_SINCOSTAB_INIT;
__device__ const double kLogPoly[5] = GLIBC239_LOG_POLY_INIT;
__device__ const double kLogPoly1[11] = GLIBC239_LOG_POLY1_INIT;
#define GLIBC_TAB(t, i) __ldg(&(t)[i])
GLIBC_HD double rn_fma(double a, double b, double c) { return __fma_rn(a, b, c); }
GLIBC_HD double rn_mul(double a, double b) { return __dmul_rn(a, b); }
GLIBC_HD double rn_add(double a, double b) { return __dadd_rn(a, b); }
GLIBC_HD double rn_sub(double a, double b) { return __dsub_rn(a, b); }
#else
static const double kLogTab[256] = GLIBC239_LOG_TAB_INIT;
static const double kSinCosTab[440] = GLIBC239_SINCOSTAB_INIT;
static const double kLogPoly[5] = GLIBC239_LOG_POLY_INIT;
static const double kLogPoly1[11] = GLIBC239_LOG_POLY1_INIT;
#define GLIBC_TAB(t, i) ((t)[i])
// volatile round trips keep the host compiler from fusing or reassociating
GLIBC_HD double rn_fma(double a, double b, double c) { return std::fma(a, b, c); }
GLIBC_HD double rn_mul(double a, double b) { volatile double r = a * b; return r; }
GLIBC_HD double rn_add(double a, double b) { volatile double r = a + b; return r; }
GLIBC_HD double rn_sub(double a, double b) { volatile double r = a - b; return r; }
#endif

// x86 fused forms: vfnmadd = -(a*b) + c, vfmsub = a*b - c (both single roundings)
GLIBC_HD double rn_fnma(double a, double b, double c) { return rn_fma(-a, b, c); }
GLIBC_HD double rn_fms(double a, double b, double c) { return rn_fma(a, b, -c); }

#if defined(__CUDA_ARCH__)
GLIBC_HD uint64_t bits(double x) { return (uint64_t)__double_as_longlong(x); }
GLIBC_HD double from_bits(uint64_t u) { return __longlong_as_double((long long)u); }
#else
GLIBC_HD uint64_t bits(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
GLIBC_HD double from_bits(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }
#endif
GLIBC_HD double abs_(double x) { return from_bits(bits(x) & 0x7fffffffffffffffULL); }
GLIBC_HD double neg_(double x) { return from_bits(bits(x) ^ 0x8000000000000000ULL); }
// vandnpd/vorpd: magnitude of v, sign of s
GLIBC_HD double copysign_(double v, double s) {
    return from_bits((bits(v) & 0x7fffffffffffffffULL) | (bits(s) & 0x8000000000000000ULL));
}

// ------------------------------------------------------------------------------- log
// __log_fma, e_log.c (LOG_TABLE_BITS 7, LOG_POLY_ORDER 6, LOG_POLY1_ORDER 12).
GLIBC_HD double log(double x) {
    const uint64_t ix = bits(x);
    // ix - LO < HI - LO with LO = asuint64(1 - 0x1p-4), HI = asuint64(1 + 0x1.09p-4)
    if (ix + 0xc012000000000000ULL <= 0x308ffffffffffULL) {
        if (ix == 0x3ff0000000000000ULL) return 0.0;
        const double* B = kLogPoly1;
        const double r = rn_sub(x, 1.0);
        // y = r3 * (B[1] + r B[2] + r2 B[3] + r3 (B[4] + r B[5] + r2 B[6]
        //         + r3 (B[7] + r B[8] + r2 B[9] + r3 B[10])))
        double p2 = rn_fma(r, GLIBC_TAB(B, 2), GLIBC_TAB(B, 1));
        double p5 = rn_fma(r, GLIBC_TAB(B, 5), GLIBC_TAB(B, 4));
        double p8 = rn_fma(r, GLIBC_TAB(B, 8), GLIBC_TAB(B, 7));
        const double r2 = rn_mul(r, r);
        p2 = rn_fma(r2, GLIBC_TAB(B, 3), p2);
        p5 = rn_fma(r2, GLIBC_TAB(B, 6), p5);
        const double r3 = rn_mul(r, r2);
        double p = rn_fma(r2, GLIBC_TAB(B, 9), p8);
        p = rn_fma(r3, GLIBC_TAB(B, 10), p);
        p = rn_fma(p, r3, p5);
        p = rn_fma(p, r3, p2);
        // w = r 2^27; rhi = r + w - w; rlo = r - rhi
        const double rw = rn_fma(r, GLIBC239_kTwo27, r);
        const double rhi = rn_fnma(GLIBC239_kTwo27, r, rw);
        const double b0 = GLIBC_TAB(B, 0);
        const double rhi2 = rn_mul(rhi, rhi);
        const double rlo = rn_sub(r, rhi);
        const double hi = rn_fma(rhi2, b0, r);          // hi = r + rhi^2 B[0]
        const double rmhi = rn_sub(r, hi);
        const double rsum = rn_add(r, rhi);
        double lo = rn_fma(rhi2, b0, rmhi);             // lo = r - hi + w
        const double b0rlo = rn_mul(b0, rlo);
        lo = rn_fma(b0rlo, rsum, lo);                   // lo += B[0] rlo (rhi + r)
        const double y = rn_fma(p, r3, lo);             // y = r3 P + lo
        return rn_add(hi, y);                           // y += hi
    }
    // x = 2^k z, z in [OFF, 2 OFF), OFF = 0x3fe6000000000000
    const uint64_t tmp = ix - 0x3fe6000000000000ULL;
    const int i = (int)((tmp >> 45) & 0x7f);
    const int k = (int)((int64_t)tmp >> 52);
    const double z = from_bits(ix - (tmp & 0xfff0000000000000ULL));
    const double kd = (double)k;
    const double invc = GLIBC_TAB(kLogTab, 2 * i), logc = GLIBC_TAB(kLogTab, 2 * i + 1);
    const double* A = kLogPoly;
    const double w = rn_fma(kd, GLIBC239_kLn2hi, logc);      // w = kd Ln2hi + logc
    const double r = rn_fma(z, invc, GLIBC239_kMinusOne);    // r = fma(z, invc, -1)
    const double q12 = rn_fma(r, GLIBC_TAB(A, 2), GLIBC_TAB(A, 1));
    const double hi = rn_add(r, w);                          // hi = w + r
    const double r2 = rn_mul(r, r);
    double lo = rn_add(rn_sub(w, hi), r);                    // lo = w - hi + r
    lo = rn_fma(kd, GLIBC239_kLn2lo, lo);                    //    + kd Ln2lo
    const double r3 = rn_mul(r, r2);
    double q34 = rn_fma(r, GLIBC_TAB(A, 4), GLIBC_TAB(A, 3));
    lo = rn_fma(r2, GLIBC_TAB(A, 0), lo);                    // lo + r2 A[0]
    q34 = rn_fma(q34, r2, q12);                              // A[1] + r A[2] + r2 (A[3] + r A[4])
    const double y = rn_fma(r3, q34, lo);
    return rn_add(y, hi);
}

// ---------------------------------------------------------------------------- sincos
// __sincos_fma, s_sincos.c. T[4 i .. 4 i + 3] = {sn, ssn, cs, ccs} of i/128.
struct TabRow {
    double sn, ssn, cs, ccs;
};
GLIBC_HD TabRow tab_row(int base) {
    return {GLIBC_TAB(kSinCosTab, base), GLIBC_TAB(kSinCosTab, base + 1),
            GLIBC_TAB(kSinCosTab, base + 2), GLIBC_TAB(kSinCosTab, base + 3)};
}
// u.x = big + |x|; xr = |x| - (u.x - big); table index = low word of u.x, times 4
GLIBC_HD int split_big(double ax, double* xr) {
    const double u = rn_add(ax, GLIBC239_kBig);
    *xr = rn_sub(ax, rn_sub(u, GLIBC239_kBig));
    return (int)((uint32_t)bits(u) << 2);
}
// TAYLOR_SIN(xx, a, da) = a + ((POLYNOMIAL(xx) a - 0.5 da) xx + da); `da_zero` is the
// da = 0 build (gcc folded "- 0.5*0" into "+ (-0.0)" and "+ 0" into an fma with 0)
GLIBC_HD double taylor_poly(double xx) {
    double p = rn_fma(xx, GLIBC239_kS5, GLIBC239_kS4);
    p = rn_fma(xx, p, GLIBC239_kS3);
    p = rn_fma(xx, p, GLIBC239_kS2);
    return rn_fma(xx, p, GLIBC239_kS1);
}
GLIBC_HD double taylor_sin(double a, double da) {
    const double xx = rn_mul(a, a);
    const double p = rn_fms(taylor_poly(xx), a, rn_mul(da, GLIBC239_kHalf));
    return rn_add(a, rn_fma(xx, p, da));
}
GLIBC_HD double taylor_sin_da_zero(double a) {
    const double xx = rn_mul(a, a);
    const double p = rn_fma(a, taylor_poly(xx), -0.0);
    return rn_add(a, rn_fma(xx, p, 0.0));
}
// sn3 + xx sn5 and cs4 + xx cs6 (both built as fma(xx, c_high, c_low))
GLIBC_HD double sn_poly(double xx) { return rn_fma(xx, GLIBC239_kSn5, GLIBC239_kSn3); }
GLIBC_HD double cs_poly(double xx) {
    return rn_fma(rn_fma(xx, GLIBC239_kCs6, GLIBC239_kCs4), xx, GLIBC239_kHalf);
}
// do_sin body after the table split: s = x + (dx + x xx (sn3 + xx sn5));
// c = x dx + xx (cs2 + xx (cs4 + xx cs6)); cor = (ssn + s ccs - sn c) + cs s; sn + cor
GLIBC_HD double do_sin_core(double xr, double dx, const TabRow& t) {
    const double xx = rn_mul(xr, xr);
    const double s = rn_add(rn_fma(rn_mul(xx, xr), sn_poly(xx), dx), xr);
    const double c = rn_fma(dx, xr, rn_mul(xx, cs_poly(xx)));
    double cor = rn_fma(s, t.ccs, t.ssn);
    cor = rn_fnma(c, t.sn, cor);
    cor = rn_fma(s, t.cs, cor);
    return rn_add(cor, t.sn);
}
// do_cos body: x = xr + dx; s = x + x xx (sn3 + xx sn5); c = xx (cs2 + ...);
// cor = (ccs - s ssn - cs c) - sn s; cs + cor
GLIBC_HD double do_cos_core(double xr, double dx, const TabRow& t) {
    const double x = rn_add(dx, xr);
    const double xx = rn_mul(x, x);
    const double s = rn_fma(rn_mul(x, xx), sn_poly(xx), x);
    const double c = rn_mul(xx, cs_poly(xx));
    double cor = rn_fnma(t.ssn, s, t.ccs);
    cor = rn_fnma(c, t.cs, cor);
    cor = rn_fnma(s, t.sn, cor);
    return rn_add(cor, t.cs);
}

GLIBC_HD void sincos(double x, double* sinx, double* cosx) {
    const uint32_t k = (uint32_t)(bits(x) >> 32) & 0x7fffffffu;
    const double ax = abs_(x);
    if (k <= 0x400368fcu) {
        if (k <= 0x3e3fffffu) {  // |x| < 2^-27: sin x = x, cos x = 1
            *sinx = x;
            *cosx = 1.0;
            return;
        }
        if (k <= 0x3feb5fffu) {  // |x| < 0.855469: do_sin(x, 0), do_cos(x, 0)
            double xr;
            const TabRow t = tab_row(split_big(ax, &xr));
            if (GLIBC239_kTaylorMax > ax) {
                *sinx = taylor_sin_da_zero(x);
            } else {
                const double dx = (x > 0.0) ? 0.0 : -0.0;  // do_sin: x <= 0 -> dx = -dx
                *sinx = copysign_(do_sin_core(xr, dx, t), x);
            }
            const double dxc = (x < 0.0) ? -0.0 : 0.0;     // do_cos: x < 0 -> dx = -dx
            *cosx = do_cos_core(xr, dxc, t);
            return;
        }
        // |x| < 2.426265: y = hp0 - |x|; a = y + hp1; da = (y - a) + hp1;
        // sin = copysign(do_cos(a, da), x); cos = do_sin(a, da)
        const double y = rn_sub(GLIBC239_kHp0, ax);
        const double a = rn_add(y, GLIBC239_kHp1);
        const double da = rn_add(rn_sub(y, a), GLIBC239_kHp1);
        const double aa = abs_(a);
        double xr;
        const TabRow t = tab_row(split_big(aa, &xr));
        *sinx = copysign_(do_cos_core(xr, (0.0 > a) ? neg_(da) : da, t), x);
        if (GLIBC239_kTaylorMax > aa)
            *cosx = taylor_sin(a, da);
        else
            *cosx = copysign_(do_sin_core(xr, (a <= 0.0) ? neg_(da) : da, t), a);
        return;
    }
    // 2.426265 <= |x| < 105414350: reduce_sincos, then do_sin / do_cos of (a, da)
    const double t = rn_fma(x, GLIBC239_kHpInv, GLIBC239_kToInt);
    const double xn = rn_sub(t, GLIBC239_kToInt);
    const int n = (int)(bits(t) & 3);
    double y = rn_fnma(xn, GLIBC239_kMp1, x);
    y = rn_fnma(xn, GLIBC239_kMp2, y);
    const double t2 = rn_fnma(xn, GLIBC239_kPp3, y);          // t2 = y - xn pp3
    double db = rn_fnma(xn, GLIBC239_kPp3, rn_sub(y, t2));    // db = (y - t2) - xn pp3
    double a = rn_fnma(xn, GLIBC239_kPp4, t2);                // b = t2 - xn pp4
    double da = rn_add(db, rn_fnma(xn, GLIBC239_kPp4, rn_sub(t2, a)));
    if (n == 1 || n == 2) {
        a = neg_(a);
        da = neg_(da);
    }
    double* to_sin = (n & 1) ? cosx : sinx;  // do_sin(a, da) lands here
    double* to_cos = (n & 1) ? sinx : cosx;  // (n & 2 ? -1 : 1) do_cos(a, da) here
    const double aa = abs_(a);
    double xr;
    const TabRow tr = tab_row(split_big(aa, &xr));
    if (GLIBC239_kTaylorMax > aa)
        *to_sin = taylor_sin(a, da);
    else
        *to_sin = copysign_(do_sin_core(xr, (0.0 >= a) ? neg_(da) : da, tr), a);
    double c = do_cos_core(xr, (a < 0.0) ? neg_(da) : da, tr);
    *to_cos = (n & 2) ? neg_(c) : c;
}

}  // namespace glibc239
