// sa_fft_cta.cuh -- CTA-cooperative register FFT for the standalone transform
// kernels (reference freqtransform.py:47-116 fft_forward / fft_inverse /
// dct_forward / dct_inverse), power-of-two complex lengths N = 256 .. 2048.
//
// The warp-per-row kernels (sa_fft.cuh) keep a series and its Stockham
// ping-pong buffer in shared memory: 2 x 16 KB per row at L = 2048, ~6 rows
// per SM, latency bound.  Here T = N / 8 threads share one row:
//
//   * thread t holds the 8 points t + m T (m < 8) in registers.  Every
//     Stockham pass of radix R in {8, 4, 2} reads exactly those points (its
//     8 / R butterflies j = t + b T take inputs j + r N / R), and the LAST
//     pass leaves output t + m T in v[m] again -- so loads from / stores to
//     global memory are coalesced 16-byte accesses with no staging;
//   * between passes the points move through ONE shared buffer of N complex
//     values (read-all / barrier / write-all), so a row needs 16 N bytes of
//     shared memory instead of 32 N: 14 rows per SM by shared memory;
//   * pass 0 (stride-8 outputs) stores XOR-swizzled (i ^ ((i >> 3) & 7)),
//     which pass 1's reads undo -- no bank conflicts in any pass.
//
// Twiddles W_{Ns R}^{r k} come from the W_L table (one load per butterfly,
// W^2k, W^4k by squaring as in sa_fft.cuh).  The real-input split / fold,
// DC / Nyquist pins and the DCT's Makhoul permutation are the same formulas
// as rfft_any / irfft_any / dct2_any / dct3_any.
#pragma once
#include "sa_fft.cuh"

namespace sa {

__device__ __forceinline__ int cta_swz(int i) { return i ^ ((i >> 3) & 7); }

// Pass plan of N = 2^LGN: radix-8 passes, then one radix-4 / radix-2 pass
// for LGN % 3 = 2 / 1.  Compile-time so every index below is static.
template <int LGN>
struct CtaPlan {
    static constexpr int N = 1 << LGN, T = N / 8;
    static constexpr int N8 = LGN / 3, REM = LGN % 3;
    static constexpr int NP = N8 + (REM ? 1 : 0);
    __host__ __device__ static constexpr int lr(int p) { return p < N8 ? 3 : REM; }
    __host__ __device__ static constexpr int lns(int p) { return p == 0 ? 0 : lns(p - 1) + lr(p - 1); }
    __host__ __device__ static constexpr int nb(int p) { return 8 >> lr(p); }  // butterflies per thread
    // first twiddle slot of pass p (pass 0 has none)
    __host__ __device__ static constexpr int slot(int p) { return p <= 1 ? 0 : slot(p - 1) + nb(p - 1); }
    static constexpr int NTW = slot(NP);  // <= 6
};

// The W^k of every (twiddled pass, butterfly) of thread t: the same for all
// rows, loaded once per kernel (tw: W_L table, N | L, L = 2^LGL).
template <int LGN>
__device__ __forceinline__ void cta_twiddles(double2 (&w)[8], int t, const double2* __restrict__ tw, int lgL) {
    using P = CtaPlan<LGN>;
#pragma unroll
    for (int p = 1; p < P::NP; ++p) {
        const int Ns = 1 << P::lns(p);
        const int tstep = 1 << (lgL - P::lns(p) - P::lr(p));  // L / (Ns R)
#pragma unroll
        for (int b = 0; b < P::nb(p); ++b) w[P::slot(p) + b] = __ldg(&tw[((t + b * P::T) & (Ns - 1)) * tstep]);
    }
}

// Radix-R butterflies of one pass on the thread's 8 points (in place in v);
// w1: this butterfly's W^k (unused for Ns == 1).
template <int R, bool TW>
__device__ __forceinline__ void cta_butterfly(double2 (&v)[8], int b, double2 w1) {
    constexpr int B = 8 / R;
    double2 u[R];
#pragma unroll
    for (int r = 0; r < R; ++r) u[r] = v[b + B * r];
    if (TW) {
        if (R == 2) {
            u[1] = cmul(u[1], w1);
        } else {
            const double2 w2 = cmul(w1, w1);
            const double2 w3 = cmul(w1, w2);
            u[1] = cmul(u[1], w1);
            u[2] = cmul(u[2], w2);
            u[3] = cmul(u[3], w3);
            if (R == 8) {
                const double2 w4 = cmul(w2, w2);
                u[4] = cmul(u[4], w4);
                u[5] = cmul(u[5], cmul(w1, w4));
                u[6] = cmul(u[6], cmul(w2, w4));
                u[7] = cmul(u[7], cmul(w3, w4));
            }
        }
    }
    if (R == 2) dft2<false>(u);
    if (R == 4) dft4<false>(u);
    if (R == 8) dft8<false>(u);
#pragma unroll
    for (int r = 0; r < R; ++r) v[b + B * r] = u[r];
}

// Store v[b + B r] (output r of butterfly b of a radix-R pass, stride
// Ns = 2^LNS) at its Stockham position; pass 0 stores swizzled.
template <int R, int LNS, int T>
__device__ __forceinline__ void cta_store(const double2 (&v)[8], double2* buf, int t) {
    constexpr int B = 8 / R;
    constexpr int LR = R == 8 ? 3 : (R == 4 ? 2 : 1);
    constexpr int Ns = 1 << LNS;
#pragma unroll
    for (int b = 0; b < B; ++b) {
        const int j = t + b * T;
        const int k = j & (Ns - 1);
        const int base = ((j >> LNS) << (LNS + LR)) + k;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int i = base + r * Ns;
            buf[LNS == 0 ? cta_swz(i) : i] = v[b + B * r];
        }
    }
}

template <int LGN, int P0>
__device__ __forceinline__ void cta_pass(double2 (&v)[8], double2* buf, int t, const double2 (&w)[8]) {
    using P = CtaPlan<LGN>;
    constexpr int LR = P::lr(P0), R = 1 << LR, LNS = P::lns(P0);
#pragma unroll
    for (int b = 0; b < 8 / R; ++b) cta_butterfly<R, (P0 > 0)>(v, b, P0 > 0 ? w[P::slot(P0) + b] : make_double2(1.0, 0.0));
    if (P0 == P::NP - 1) return;
    __syncthreads();  // every thread has read the previous pass's buffer
    cta_store<R, LNS, P::T>(v, buf, t);
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        const int i = t + m * P::T;
        v[m] = buf[P0 == 0 ? cta_swz(i) : i];
    }
}

// Forward N-point FFT (N = 2^LGN = 8 T, 256 <= N <= 2048) of the points the
// CTA holds in registers (v[m] = z[t + m T]); on return v[m] = Z[t + m T].
// w: cta_twiddles.  buf: N complex of shared memory, free on entry (the
// caller has barriered its own earlier readers), in use on return until the
// caller's next barrier.
template <int LGN>
__device__ __forceinline__ void cta_fft(double2 (&v)[8], double2* buf, int t, const double2 (&w)[8]) {
    using P = CtaPlan<LGN>;
    cta_pass<LGN, 0>(v, buf, t, w);
    if (P::NP > 1) cta_pass<LGN, (P::NP > 1 ? 1 : 0)>(v, buf, t, w);
    if (P::NP > 2) cta_pass<LGN, (P::NP > 2 ? 2 : 0)>(v, buf, t, w);
    if (P::NP > 3) cta_pass<LGN, (P::NP > 3 ? 3 : 0)>(v, buf, t, w);
}

}  // namespace sa
