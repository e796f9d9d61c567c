// sa_fft.cuh -- warp-level FP64 real FFT / inverse in shared memory.
//
// Replaces pocketfft's np.fft.rfft / irfft on the augmentation path
// (reference freqaugment.py:40-47, freqtransform.py:101-116).  One warp
// transforms one series that already sits in shared memory:
//
//   rfft(L = 2M):  view x as M complex samples z[n] = x[2n] + i x[2n+1]
//                  (no data movement), M-point complex FFT by Stockham
//                  autosort passes of radix 8/4/2 ping-ponging between two
//                  smem buffers, then the split step
//                  X[k] = E[k] + W_L^k O[k], k = 0..M.
//   irfft:         the inverse split, then the SAME forward passes on the
//                  conjugate (IFFT(Z) = conj(FFT(conj Z))), 1/M scaling,
//                  result read back as the real series in place.
//
// Twiddles come from a per-length table tw[k] = exp(-2*pi*i*k/L), k < L,
// computed on the host in long double (correctly rounded) and cached.
// Parity with pocketfft is to tolerance (FFT rounding differs), so FMAs are
// used explicitly here even though the rest of the TU is built -fmad=false.
#pragma once
#include <stdint.h>

namespace sa {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ double2 rot90(double2 a) {
    return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

template <bool INV>
__device__ __forceinline__ void dft2(double2* v) {
    double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
}

template <bool INV>
__device__ __forceinline__ void dft4(double2* v) {
    double2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
    double2 b0 = cadd(v[1], v[3]), b1 = rot90<INV>(csub(v[1], v[3]));
    v[0] = cadd(a0, b0);
    v[2] = csub(a0, b0);
    v[1] = cadd(a1, b1);
    v[3] = csub(a1, b1);
}

template <bool INV>
__device__ __forceinline__ void dft8(double2* v) {
    const double h = 0.70710678118654752440;
    double2 e[4] = {v[0], v[2], v[4], v[6]};
    double2 o[4] = {v[1], v[3], v[5], v[7]};
    dft4<INV>(e);
    dft4<INV>(o);
    // o[k] *= W8^k (forward W8 = exp(-i*pi/4))
    double2 o1 = o[1], o3 = o[3];
    o[1] = INV ? make_double2((o1.x - o1.y) * h, (o1.x + o1.y) * h)
               : make_double2((o1.x + o1.y) * h, (o1.y - o1.x) * h);
    o[2] = rot90<INV>(o[2]);
    o[3] = INV ? make_double2(-(o3.x + o3.y) * h, (o3.x - o3.y) * h)
               : make_double2((o3.y - o3.x) * h, -(o3.x + o3.y) * h);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[k] = cadd(e[k], o[k]);
        v[k + 4] = csub(e[k], o[k]);
    }
}

// One Stockham pass of radix R over M points: src -> dst.
// tw: exp(-2 pi i q / L), L = 2M; W_{Ns R}^{rk} = tw[r k (L / (Ns R))].
template <int R, bool INV>
__device__ __forceinline__ void stockham_pass(const double2* __restrict__ src, double2* __restrict__ dst,
                                              int M, int Ns, const double2* __restrict__ tw, int L,
                                              int lane) {
    const int Q = M / R;
    const int tstep = L / (Ns * R);
    for (int j = lane; j < Q; j += 32) {
        int k = j & (Ns - 1);
        double2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = src[j + r * Q];
        if (Ns > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) {
                double2 w = __ldg(&tw[r * k * tstep]);
                if (INV) w.y = -w.y;
                v[r] = cmul(v[r], w);
            }
        }
        if (R == 2) dft2<INV>(v);
        if (R == 4) dft4<INV>(v);
        if (R == 8) dft8<INV>(v);
        int base = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) dst[base + r * Ns] = v[r];
    }
    __syncwarp();
}

// M-point complex FFT (M a power of two), data in a; b is scratch.
// Returns the buffer holding the result.
template <bool INV>
__device__ double2* fft_pow2(double2* a, double2* b, int M, const double2* tw, int L, int lane) {
    int Ns = 1;
    double2* src = a;
    double2* dst = b;
    while (Ns < M) {
        int rem = M / Ns;
        if (rem >= 8 && rem != 16) {  // 16 = 4 x 4 keeps passes balanced
            stockham_pass<8, INV>(src, dst, M, Ns, tw, L, lane);
            Ns *= 8;
        } else if (rem >= 4) {
            stockham_pass<4, INV>(src, dst, M, Ns, tw, L, lane);
            Ns *= 4;
        } else {
            stockham_pass<2, INV>(src, dst, M, Ns, tw, L, lane);
            Ns *= 2;
        }
        double2* t = src;
        src = dst;
        dst = t;
    }
    return src;
}

// rfft of x (length L = 2M, in buffer xa viewed as complex) into X[0..M]
// (M + 1 complex).  xb is scratch of the same capacity.  Returns the buffer
// holding X (one of xa / xb); the other is free afterwards.
__device__ __forceinline__ double2* rfft_warp(double* xa, double* xb, int L, const double2* tw, int lane) {
    const int M = L >> 1;
    double2* za = reinterpret_cast<double2*>(xa);
    double2* zb = reinterpret_cast<double2*>(xb);
    double2* Z = fft_pow2<false>(za, zb, M, tw, L, lane);
    double2* X = (Z == za) ? zb : za;
    for (int k = lane; k <= M; k += 32) {
        double2 zk = Z[k == M ? 0 : k];
        double2 zc = Z[k == 0 ? 0 : M - k];
        double er = 0.5 * (zk.x + zc.x), ei = 0.5 * (zk.y - zc.y);
        double orr = 0.5 * (zk.y + zc.y), oi = -0.5 * (zk.x - zc.x);
        double2 w = __ldg(&tw[k]);
        double2 o = cmul(make_double2(orr, oi), w);
        X[k] = make_double2(er + o.x, ei + o.y);
    }
    __syncwarp();
    if (lane == 0) {
        X[0].y = 0.0;
        X[M].y = 0.0;
    }
    __syncwarp();
    return X;
}

// irfft of X[0..M] (in buffer X) to a real series of length L = 2M.
// Returns the buffer holding the series (one of X / other).
__device__ __forceinline__ double* irfft_warp(double2* X, double2* other, int L, const double2* tw, int lane) {
    const int M = L >> 1;
    // inverse split; store conj(Z) so the forward passes compute conj(IFFT)
    for (int k = lane; k < M; k += 32) {
        double2 xk = X[k];
        double2 xc = X[M - k];
        if (k == 0) { xk.y = 0.0; xc.y = 0.0; }  // irfft ignores im of DC / Nyquist
        xc.y = -xc.y;
        double er = 0.5 * (xk.x + xc.x), ei = 0.5 * (xk.y + xc.y);
        double dr = 0.5 * (xk.x - xc.x), di = 0.5 * (xk.y - xc.y);
        double2 w = __ldg(&tw[k]);
        w.y = -w.y;
        double2 o = cmul(make_double2(dr, di), w);
        other[k] = make_double2(er - o.y, -(ei + o.x));
    }
    __syncwarp();
    double2* Z = fft_pow2<false>(other, X, M, tw, L, lane);
    const double s = 1.0 / (double)M;
    for (int k = lane; k < M; k += 32) {
        double2 z = Z[k];
        Z[k] = make_double2(z.x * s, -(z.y * s));
    }
    __syncwarp();
    return reinterpret_cast<double*>(Z);
}

}  // namespace sa
