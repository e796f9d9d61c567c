// sa_log1p.h -- log1p with the rounding of the reference's libm.
//
// numpy's ziggurat tail (random_standard_normal, idx 0) evaluates
// npy_log1p = the C library's log1p.  On the reference's platform (x86_64,
// glibc 2.39, the CPU having FMA) that is the fdlibm algorithm (argument
// reduction to 1+f in [sqrt(2)/2, sqrt(2)), s = f/(2+f), a degree-7
// polynomial in s^2 with the Lp1..Lp7 coefficients) with the polynomial in
// Estrin form and the multiply-add pairs the compiler fuses into FMAs.  It is
// not correctly rounded (it differs from the correctly rounded log1p in ~7% of
// arguments), so no other log1p -- CUDA's included -- reproduces its bits; this
// restatement does, and every fused multiply-add below is written as an
// explicit fma() (the translation units are built with -fmad=false /
// -ffp-contract=off, so no other operation is contracted).
//
// Pinned by tests/test_log1p_pin.py: bitwise equal to the host libm's log1p on
// 2e7 arguments per domain (the tail's log1p(-u), u = k 2^-53; tiny, positive
// and random-bit arguments), on the CPU (this header compiled by gcc) and on
// the device (tests/csrc/rng_probe.cu).
#pragma once
#include <stdint.h>
#include <math.h>
#if !defined(__CUDACC__)
#include <string.h>
#endif

#if defined(__CUDACC__)
#define SA_L1P_FN __host__ __device__ __forceinline__
#else
#define SA_L1P_FN static inline
#endif

SA_L1P_FN int32_t sa_l1p_hi(double x) {
#if defined(__CUDA_ARCH__)
    return __double2hiint(x);
#else
    uint64_t b;
    memcpy(&b, &x, 8);
    return (int32_t)(b >> 32);
#endif
}

SA_L1P_FN double sa_l1p_with_hi(double x, int32_t h) {
#if defined(__CUDA_ARCH__)
    return __hiloint2double(h, __double2loint(x));
#else
    uint64_t b;
    memcpy(&b, &x, 8);
    b = (b & 0xffffffffull) | ((uint64_t)(uint32_t)h << 32);
    memcpy(&x, &b, 8);
    return x;
#endif
}

SA_L1P_FN double sa_log1p(double x) {
    const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
    const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
                 Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
                 Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
                 Lp7 = 1.479819860511658591e-01;
    double f = 0.0, c = 0.0, u;
    const int32_t hx = sa_l1p_hi(x), ax = hx & 0x7fffffff;
    int32_t k = 1, hu = 0;
    if (hx < 0x3FDA827A) {  // x < 0.41422
        if (ax >= 0x3ff00000) return x == -1.0 ? -INFINITY : NAN;  // x <= -1
        if (ax < 0x3e200000) {                                      // |x| < 2^-29
            if (ax < 0x3c900000) return x;                          // |x| < 2^-54
            return fma(-(x * x), 0.5, x);
        }
        if (hx > 0 || hx <= (int32_t)0xbfd2bec3) {  // -0.2929 < x < 0.41422
            k = 0;
            f = x;
            hu = 1;
        }
    }
    if (hx >= 0x7ff00000) return x + x;
    if (k != 0) {
        if (hx < 0x43400000) {
            u = 1.0 + x;
            hu = sa_l1p_hi(u);
            k = (hu >> 20) - 1023;
            c = (k > 0) ? 1.0 - (u - x) : x - (u - 1.0);  // correction term
            c /= u;
        } else {
            u = x;
            hu = sa_l1p_hi(u);
            k = (hu >> 20) - 1023;
            c = 0.0;
        }
        hu &= 0x000fffff;
        if (hu < 0x6a09e) {
            u = sa_l1p_with_hi(u, hu | 0x3ff00000);  // normalise u
        } else {
            k += 1;
            u = sa_l1p_with_hi(u, hu | 0x3fe00000);  // normalise u/2
            hu = (0x00100000 - hu) >> 2;
        }
        f = u - 1.0;
    }
    const double dk = (double)k;
    const double hfsq = (f * 0.5) * f;
    if (hu == 0) {  // |f| < 2^-20
        if (f == 0.0) {
            if (k == 0) return 0.0;
            c = fma(dk, ln2_lo, c);
            return fma(dk, ln2_hi, c);
        }
        const double R = fma(-f, 0.66666666666666666, 1.0) * hfsq;
        if (k == 0) return f - R;
        return fma(dk, ln2_hi, -((R - fma(dk, ln2_lo, c)) - f));
    }
    const double s = f / (2.0 + f);
    const double z = s * s;
    const double z2 = z * z, R2 = fma(z, Lp3, Lp2), z4 = z2 * z2, R3 = fma(z, Lp5, Lp4);
    const double z6 = z2 * z4, R4 = fma(z, Lp7, Lp6);
    const double R = fma(z6, R4, fma(z4, R3, fma(z, Lp1, z2 * R2)));
    const double w = s * (hfsq + R);
    if (k == 0) return f - (hfsq - w);
    return fma(dk, ln2_hi, -((hfsq - (fma(dk, ln2_lo, c) + w)) - f));
}
