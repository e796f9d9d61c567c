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
// General lengths (pocketfft handles any L): the complex length N (= L/2
// packed for even L, = L for odd L, whose real input is complexified) is
// factored on the host into radix-8/4/2 passes followed by one generic pass
// per remaining prime factor (each output of a generic pass is a direct
// R-term sum with one twiddle lookup per term).
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

// 16-point DFT as 4 x 4: n = n1 + 4 n2, k = 4 k1 + k2.  DFT4 over n2 for each
// n1, multiply by W16^(n1 k2), DFT4 over n1 for each k2.
template <bool INV>
__device__ __forceinline__ void dft16(double2* v) {
    double2 y[16];  // y[4 * n1 + k2]
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) {
        double2 t[4] = {v[n1], v[n1 + 4], v[n1 + 8], v[n1 + 12]};
        dft4<INV>(t);
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) y[4 * n1 + k2] = t[k2];
    }
    // W16^e, e = n1 * k2 in {1, 2, 3, 4, 6, 9}
    const double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;  // cos, sin pi/8
    const double h = 0.70710678118654752440;
    const double sg = INV ? 1.0 : -1.0;  // forward: exp(-i ...)
    const double2 w1 = make_double2(c1, sg * s1), w2 = make_double2(h, sg * h), w3 = make_double2(s1, sg * c1);
    const double2 w6 = make_double2(-h, sg * h), w9 = make_double2(-c1, -sg * s1);
    y[5] = cmul(y[5], w1);
    y[6] = cmul(y[6], w2);
    y[7] = cmul(y[7], w3);
    y[9] = cmul(y[9], w2);
    y[10] = rot90<INV>(y[10]);  // W16^4
    y[11] = cmul(y[11], w6);
    y[13] = cmul(y[13], w3);
    y[14] = cmul(y[14], w6);
    y[15] = cmul(y[15], w9);
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
        double2 t[4] = {y[k2], y[4 + k2], y[8 + k2], y[12 + k2]};
        dft4<INV>(t);
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) v[4 * k1 + k2] = t[k1];
    }
}

// One Stockham pass of radix R (2, 4, 8, 16) over M points: src -> dst, for
// Ns = 2^lns (the power-of-two passes run first, so Ns is a power of two).
// tw: exp(-2 pi i q / L); W_{Ns R}^{rk} = tw[r k tstep], tstep = L / (Ns R).
// Twiddles: W^k, W^2k, W^4k are loaded, the odd powers multiplied out.
// Swizzled intermediate: the first pass writes dst[R j + r] (stride R across
// lanes -> an R-way shared-memory bank conflict).  That buffer (read only by
// the second pass) is stored at i ^ ((i >> log2 R) & (R - 1)), which spreads
// each 8-lane phase over distinct banks for both the writes and the reads.
struct Swz {
    int sh, mask;  // mask == 0: identity
    __device__ __forceinline__ int operator()(int i) const { return i ^ ((i >> sh) & mask); }
};

// FIN (irfft's last pass): outputs are stored as conj(v) * fin_s and OR-ed
// into *fin_bad when non-finite (the irfft scaling loop, fused).
__device__ __forceinline__ bool fin_bad(double v);
template <int R, bool INV, bool FIN = false>
__device__ __forceinline__ void stockham_pass(const double2* __restrict__ src, double2* __restrict__ dst,
                                              int M, int lns, const double2* __restrict__ tw, int tstep,
                                              int lane, Swz sin = {0, 0}, Swz sout = {0, 0}, double fin_s = 1.0,
                                              bool* fin_bad_out = nullptr) {
    const int Q = M / R;
    const int Ns = 1 << lns;
#pragma unroll 2
    for (int j = lane; j < Q; j += 32) {
        const int k = j & (Ns - 1);
        double2 v[R];
        // the swizzle term of j + rQ is the same for every r (fft_any only
        // swizzles when Q is a multiple of R_prev^2), so it is applied once
        const double2* sj = src + sin(j);
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = sj[r * Q];
        if (Ns > 1) {
            double2 w1 = __ldg(&tw[k * tstep]);
            if (INV) w1.y = -w1.y;
            if (R == 2) {
                v[1] = cmul(v[1], w1);
            } else {
                // one table load per butterfly: W^2k, W^4k (W^8k) by squaring
                // (the table sits in L2 -- shared memory holds the series)
                const double2 w2 = cmul(w1, w1);
                const double2 w3 = cmul(w1, w2);
                v[1] = cmul(v[1], w1);
                v[2] = cmul(v[2], w2);
                v[3] = cmul(v[3], w3);
                if (R >= 8) {
                    const double2 w4 = cmul(w2, w2);
                    v[4] = cmul(v[4], w4);
                    v[5] = cmul(v[5], cmul(w1, w4));
                    v[6] = cmul(v[6], cmul(w2, w4));
                    v[7] = cmul(v[7], cmul(w3, w4));
                    if (R == 16) {
                        const double2 w8 = cmul(w4, w4);
#pragma unroll
                        for (int r = 1; r < 8; ++r) {
                            const double2 wr = r == 1 ? w1 : r == 2 ? w2 : r == 3 ? w3 : r == 4 ? w4
                                             : r == 5 ? cmul(w1, w4) : r == 6 ? cmul(w2, w4) : cmul(w3, w4);
                            v[8 + r] = cmul(v[8 + r], cmul(wr, w8));
                        }
                        v[8] = cmul(v[8], w8);
                    }
                }
            }
        }
        if (R == 2) dft2<INV>(v);
        if (R == 4) dft4<INV>(v);
        if (R == 8) dft8<INV>(v);
        if (R == 16) dft16<INV>(v);
        const int base = ((j >> lns) << (lns + (R == 16 ? 4 : (R == 8 ? 3 : (R == 4 ? 2 : 1))))) + k;
        // output swizzle only on pass 0 (Ns == 1, base a multiple of R): one
        // XOR term for the whole butterfly
        const int xo = (base >> sout.sh) & sout.mask;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (FIN) {
                const double2 o = make_double2(v[r].x * fin_s, -(v[r].y * fin_s));
                *fin_bad_out |= fin_bad(o.x) | fin_bad(o.y);
                dst[(base + r * Ns) ^ xo] = o;
            } else {
                dst[(base + r * Ns) ^ xo] = v[r];
            }
        }
    }
    __syncwarp();
}

// Host-built pass plan of an N-point complex FFT (N | L).  N with a large
// prime factor uses Bluestein instead (blue = 1): the N-point DFT as a
// circular convolution of length M (a power of two >= 2N - 1), i.e. two
// M-point FFTs and a pointwise product with the precomputed FFT of the
// chirp kernel -- O(M log M) like pocketfft, instead of the O(N p) generic
// pass.  M's radix plan and tables ride along.
#define SA_FFT_MAXPASS 24
struct FftGeo {
    int32_t N;         // complex transform length
    int32_t packed;    // 1: even L, N = L/2 (real input viewed as complex)
    int32_t npass;
    int32_t blue;      // 1: Bluestein
    int32_t oddreal;   // odd L as a real transform (rfft_any): 1 paired columns, 2 Bluestein on the bins k <= L/2
    int16_t radix[SA_FFT_MAXPASS];
    int32_t M, mpass;  // Bluestein convolution length and its radix plan
    int16_t mradix[16];
    const double2* chirp;  // exp(-i pi n^2 / N), n < N
    const double2* bfft;   // FFT_M of the kernel exp(+i pi m^2 / N), circular
    const double2* twM;    // exp(-2 pi i k / M), k < M
};

// Generic radix-R Stockham pass, R an odd prime (R | N).  Output u of column
// j is the R-point DFT of the twiddled column y_r = src[j + rQ] W_N^(r k a):
// V[u] = sum_r y_r W_R^(ru).  Folding the pairs r, R - r (s_r = y_r +
// y_(R-r), d_r = y_r - y_(R-r)) gives, for the output pair u, R - u,
//   V[u]     = y_0 + sum_m s_m cos(2 pi m u / R) - i sum_m d_m sin(2 pi m u / R)
//   V[R - u] = y_0 + sum_m s_m cos(2 pi m u / R) + i sum_m d_m sin(2 pi m u / R)
// (m = 1 .. (R-1)/2): 4 real FMAs per (m, output pair) instead of 16 for the
// direct complex sums.  Step 1 twiddles and folds each column in place in
// `src` (this pass's input is scratch afterwards); step 2 accumulates four
// output pairs per work item over the folded column, cos / sin exact from the
// W_L table (index m u mod R kept incrementally).
//
// Q columns of R points; tsa = L / (Ns R), the W_{Ns R} stride in the W_L
// table (0: the columns arrive twiddled).  hl >= 0 (the last pass of the
// odd-length real transform, rfft_any): only the columns j <= (Ns - 1) / 2 are
// present, and an output index above hl = (L - 1) / 2 is stored as the
// conjugate at L - index (the spectrum of a real series is Hermitian; the
// mirrors are the columns Ns - j that were left out).
__device__ __forceinline__ void generic_pass(double2* __restrict__ src, double2* __restrict__ dst, int Q, int Ns,
                                             int R, const double2* __restrict__ tw, int L, int lane, int tsa,
                                             int hl) {
    const int tr = L / R;  // W_R stride
    const int H = (R - 1) >> 1;
    auto put = [&](int i, double re, double im) {
        if (hl >= 0 && i > hl) {
            i = L - i;
            im = -im;
        }
        dst[i] = make_double2(re, im);
    };
    for (int idx = lane; idx < Q * H; idx += 32) {
        const int j = idx % Q, m = 1 + idx / Q;
        const int ka = (j % Ns) * tsa;  // exponents r ka < L: no reduction
        double2 y1 = src[j + m * Q], y2 = src[j + (R - m) * Q];
        if (ka) {
            y1 = cmul(y1, __ldg(&tw[m * ka]));
            y2 = cmul(y2, __ldg(&tw[(R - m) * ka]));
        }
        src[j + m * Q] = cadd(y1, y2);
        src[j + (R - m) * Q] = csub(y1, y2);
    }
    __syncwarp();
    const int G = (H + 4) >> 2;  // output pairs u = 0 .. H, four per item
    if (Q * G < 32) {
        // few columns (small N, e.g. a prime length): one output pair per
        // item keeps more lanes busy; each output accumulates over m in the
        // same order as below, so the result is the same
        for (int idx = lane; idx < Q * (H + 1); idx += 32) {
            const int j = idx % Q, u = idx / Q;
            const int k = j % Ns;
            const double2 y0 = src[j];
            double2 A = make_double2(0.0, 0.0), B = make_double2(0.0, 0.0);
            int id = 0;
            for (int m = 1; m <= H; ++m) {
                const double2 sm = src[j + m * Q], dm = src[j + (R - m) * Q];
                id += u;
                id = id >= R ? id - R : id;
                const double2 w = __ldg(&tw[id * tr]);
                A.x = fma(sm.x, w.x, A.x);
                A.y = fma(sm.y, w.x, A.y);
                B.x = fma(dm.x, w.y, B.x);
                B.y = fma(dm.y, w.y, B.y);
            }
            const int o = (j - k) * R + k;
            const double re = y0.x + A.x, im = y0.y + A.y;
            put(o + u * Ns, re - B.y, im + B.x);
            if (u) put(o + (R - u) * Ns, re + B.y, im - B.x);
        }
        __syncwarp();
        return;
    }
    for (int idx = lane; idx < Q * G; idx += 32) {
        const int j = idx % Q, g0 = 4 * (idx / Q);
        const int k = j % Ns;
        const double2 y0 = src[j];
        double2 A[4], B[4];
        int id[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            A[c] = make_double2(0.0, 0.0);
            B[c] = make_double2(0.0, 0.0);
            id[c] = 0;
        }
        for (int m = 1; m <= H; ++m) {
            const double2 sm = src[j + m * Q], dm = src[j + (R - m) * Q];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                id[c] += g0 + c;  // m u mod R, u = g0 + c <= H + 3 < R
                id[c] = id[c] >= R ? id[c] - R : id[c];
                const double2 w = __ldg(&tw[id[c] * tr]);  // (cos, -sin)
                A[c].x = fma(sm.x, w.x, A[c].x);
                A[c].y = fma(sm.y, w.x, A[c].y);
                B[c].x = fma(dm.x, w.y, B[c].x);  // B = -sum d sin
                B[c].y = fma(dm.y, w.y, B[c].y);
            }
        }
        const int o = (j - k) * R + k;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int u = g0 + c;
            if (u > H) break;
            const double re = y0.x + A[c].x, im = y0.y + A[c].y;
            // -i * (-B) = (-B.y, B.x) for V[u]; its negation for V[R - u]
            put(o + u * Ns, re - B[c].y, im + B[c].x);
            if (u) put(o + (R - u) * Ns, re + B[c].y, im - B[c].x);
        }
    }
    __syncwarp();
}

// The Stockham passes of an N-point plan (radix list `radix`, npass passes)
// over a table of W_L (N | L); data in a, b is scratch; returns the buffer
// holding the result.
//
// real_last (odd composite L = P q, P the last radix; rfft_any's paired-column
// real transform): N = (P + 1) / 2 * q, the passes before the last leave the
// q-point transforms Z_c of the column pairs z_c[m] = x[2c + m P] + i x[2c + 1
// + m P]; real_unpack separates and twiddles them into the columns j <= (q -
// 1) / 2 of the last pass, which then runs on half the columns.
__device__ __forceinline__ void real_unpack(const double2* __restrict__ Z, double2* __restrict__ Y, int P, int q,
                                            const double2* __restrict__ tw, int lane) {
    const int Pp = (P + 1) >> 1, Qh = (q + 1) >> 1;
    for (int idx = lane; idx < Pp * Qh; idx += 32) {
        const int c = idx / Qh, j = idx - c * Qh;
        const double2 zj = Z[c * q + j], zc = Z[c * q + (j ? q - j : 0)];
        // F_2c = (Z[j] + conj Z[q - j]) / 2, F_2c+1 = (Z[j] - conj Z[q - j]) / 2i
        const double2 fe = make_double2(0.5 * (zj.x + zc.x), 0.5 * (zj.y - zc.y));
        const double2 fo = make_double2(0.5 * (zj.y + zc.y), -0.5 * (zj.x - zc.x));
        const int r = 2 * c;
        Y[j + r * Qh] = (r * j) ? cmul(fe, __ldg(&tw[r * j])) : fe;  // W_L^{r j}, r j < L
        if (r + 1 < P) Y[j + (r + 1) * Qh] = j ? cmul(fo, __ldg(&tw[(r + 1) * j])) : fo;
    }
    __syncwarp();
}

// ODD: the generic (odd prime) passes and the odd-length real transform are
// compiled in.  The chain kernel keeps them -- and Bluestein -- out of the
// instantiation that runs the power-of-two plans: its code generation is
// sensitive to everything inlined into it.
template <bool R16 = false, bool ODD = true>
__device__ __forceinline__ double2* fft_passes(double2* a, double2* b, int N, int npass, const int16_t* radix,
                                               const double2* tw, int L, int lane, bool real_last = false) {
    int Ns = 1;
    double2* src = a;
    double2* dst = b;
    int lns = 0;
    Swz carry = {0, 0};  // swizzle of the buffer the next pass reads
    for (int p = 0; p < npass; ++p) {
        const int R = radix[p];
        if (R == 16 || R == 8 || R == 4 || R == 2) {
            const int lr = (R == 16 ? 4 : (R == 8 ? 3 : (R == 4 ? 2 : 1)));
            const int tstep = L >> (lns + lr);  // L / (Ns R)
            // swizzle pass 0's output when pass 1 is a power-of-two pass too
            const bool swz = (p == 0 && R > 2 && R < 16 && npass > 1 && (radix[1] & (radix[1] - 1)) == 0 &&
                              (N / radix[1]) % (R * R) == 0);
            const Swz out = swz ? Swz{lr, R - 1} : Swz{0, 0};
            if (R16 && R == 16) stockham_pass<R16 ? 16 : 8, false>(src, dst, N, lns, tw, tstep, lane, carry, out);
            else if (R == 8) stockham_pass<8, false>(src, dst, N, lns, tw, tstep, lane, carry, out);
            else if (R == 4) stockham_pass<4, false>(src, dst, N, lns, tw, tstep, lane, carry, out);
            else stockham_pass<2, false>(src, dst, N, lns, tw, tstep, lane, carry, out);
            carry = out;
            lns += lr;
        } else if (ODD) {  // (plans with a generic pass run the ODD instantiations)
            if (ODD && real_last && p == npass - 1) {  // Ns = q here
                real_unpack(src, dst, R, Ns, tw, lane);
                double2* t = src;
                src = dst;
                dst = t;
                generic_pass(src, dst, (Ns + 1) >> 1, Ns, R, tw, L, lane, 0, (L - 1) >> 1);
            } else {  // (its own copy: hl = -1 folds the mirrored store away)
                generic_pass(src, dst, N / R, Ns, R, tw, L, lane, L / (Ns * R), -1);
            }
        }
        Ns *= R;
        double2* t = src;
        src = dst;
        dst = t;
    }
    return src;
}

// Bluestein: X[k] = c[k] * sum_n (x[n] c[n]) conj(c[k - n]), c[n] =
// exp(-i pi n^2 / N), evaluated as IFFT_M(FFT_M(x c) * FFT_M(conj c)) with
// IFFT(V) = conj(FFT(conj V)) / M.  a holds x (N points); a and b hold M.
__device__ __forceinline__ double2* bluestein(double2* a, double2* b, const FftGeo& g, int lane) {
    const int N = g.N, M = g.M;
    for (int n = lane; n < M; n += 32) b[n] = n < N ? cmul(a[n], __ldg(&g.chirp[n])) : make_double2(0.0, 0.0);
    __syncwarp();
    double2* Y = fft_passes<false, false>(b, a, M, g.mpass, g.mradix, g.twM, M, lane);
    for (int k = lane; k < M; k += 32) {
        const double2 v = cmul(Y[k], __ldg(&g.bfft[k]));
        Y[k] = make_double2(v.x, -v.y);
    }
    __syncwarp();
    double2* Z = fft_passes<false, false>(Y, Y == a ? b : a, M, g.mpass, g.mradix, g.twM, M, lane);
    const double inv = 1.0 / (double)M;
    for (int k = lane; k < N; k += 32) {
        const double2 z = Z[k];
        Z[k] = cmul(make_double2(z.x * inv, -z.y * inv), __ldg(&g.chirp[k]));
    }
    __syncwarp();
    return Z;
}

// N = 512 (L = 1024, the configs' length) as compile-time constants: the
// same radix-8 x 3 Stockham plan and pass-0 swizzle fft_passes runs for it,
// with every size, stride, twiddle step and swizzle folded into the code
// (no runtime pass loop or index arithmetic).  Same arithmetic, same result.
// FIN: irfft's conj / 1/N scaling and finiteness check fused into the last pass.
template <bool FIN = false>
__device__ __forceinline__ double2* fft_512(double2* a, double2* b, const double2* tw, int lane, bool* bad = nullptr) {
    constexpr int N = 512, L = 1024;
    stockham_pass<8, false>(a, b, N, 0, tw, L >> 3, lane, Swz{0, 0}, Swz{3, 7});
    stockham_pass<8, false>(b, a, N, 3, tw, L >> 6, lane, Swz{3, 7}, Swz{0, 0});
    stockham_pass<8, false, FIN>(a, b, N, 6, tw, L >> 9, lane, Swz{0, 0}, Swz{0, 0}, 1.0 / (double)N, bad);
    return b;
}

// Forward N-point complex FFT per the plan; data in a, b is scratch.
__device__ __forceinline__ bool is_fft_512(const FftGeo& g, int L) {
    return L == 1024 && !g.blue && g.N == 512 && g.npass == 3 && g.radix[0] == 8 && g.radix[1] == 8 && g.radix[2] == 8;
}

// FIN (irfft of the fft_512 plan only): see fft_512.
template <bool BLUE = true, bool R16 = false, bool FIN = false, bool ODD = true>
__device__ __forceinline__ double2* fft_any(double2* a, double2* b, const FftGeo& g, const double2* tw, int L,
                                            int lane, bool* fin_bad_out = nullptr) {
    if (BLUE && g.blue) return bluestein(a, b, g, lane);
    if (is_fft_512(g, L)) return fft_512<FIN>(a, b, tw, lane, fin_bad_out);
    // oddreal: a holds the (P + 1) / 2 * q packed column pairs (rfft_any)
    const bool odd = ODD && g.oddreal == 1;
    const int P = odd ? g.radix[g.npass - 1] : 1;
    const int N = odd ? ((P + 1) >> 1) * (g.N / P) : g.N;
    return fft_passes<R16, ODD>(a, b, N, g.npass, g.radix, tw, L, lane, odd);
}

// rfft split X[k] = E[k] + W_L^k O[k] from Z[k], Z[M - k] (rfft_any).
__device__ __forceinline__ double2 cta_split(double2 zk, double2 zc, double2 w) {
    const double er = 0.5 * (zk.x + zc.x), ei = 0.5 * (zk.y - zc.y);
    const double orr = 0.5 * (zk.y + zc.y), oi = -0.5 * (zk.x - zc.x);
    const double2 o = cmul(make_double2(orr, oi), w);
    return make_double2(er + o.x, ei + o.y);
}

// irfft fold of X[k], X[M - k] into the conjugated FFT input (irfft_any).
__device__ __forceinline__ double2 cta_fold(double2 xk, double2 xc, double2 w, bool k0) {
    if (k0) { xk.y = 0.0; xc.y = 0.0; }
    xc.y = -xc.y;
    const double er = 0.5 * (xk.x + xc.x), ei = 0.5 * (xk.y + xc.y);
    const double dr = 0.5 * (xk.x - xc.x), di = 0.5 * (xk.y - xc.y);
    w.y = -w.y;
    const double2 o = cmul(make_double2(dr, di), w);
    return make_double2(er - o.y, -(ei + o.x));
}

// Odd composite L = P q (P the plan's last radix): the P decimated series
// x[r + m P] are real, so they are transformed two at a time, z_c[m] =
// x[2c + m P] + i x[2c + 1 + m P] (the last one alone), laid out as
// u[c + m (P + 1) / 2] for the plan's first passes; the last pass separates
// the pairs and runs on half the columns (fft_passes).
__device__ __forceinline__ void oddreal_pack(const double* __restrict__ x, double2* __restrict__ u, int L, int P,
                                          int lane) {
    const int Pp = (P + 1) >> 1, Np = Pp * (L / P);
    for (int n = lane; n < Np; n += 32) {
        const int m = n / Pp, c = n - m * Pp;
        const int i = 2 * c + m * P;
        u[n] = make_double2(x[i], 2 * c + 1 < P ? x[i + 1] : 0.0);
    }
    __syncwarp();
}
// x = irfft(X) through ONE forward real transform: h[k] = Re X[k] - Im X[k]
// over the Hermitian completion (h[L - k] = Re X[k] + Im X[k]) is real; its
// transform H has Re H[t] = sum_k Re X[k] cos(2 pi k t / L) and Im H[t] =
// sum_k Im X[k] sin(2 pi k t / L), so L x[t] = Re H[t] - Im H[t] and
// L x[L - t] = Re H[t] + Im H[t].
__device__ __forceinline__ void oddreal_fold(const double2* __restrict__ X, double* __restrict__ h, int L, int lane) {
    for (int k = lane; k <= L / 2; k += 32) {
        const double2 v = X[k];
        if (k == 0) {
            h[0] = v.x;
        } else {
            h[k] = v.x - v.y;
            h[L - k] = v.x + v.y;
        }
    }
    __syncwarp();
}
__device__ __forceinline__ bool fin_bad(double v);
__device__ __forceinline__ bool oddreal_unfold(const double2* __restrict__ H, double* __restrict__ out, int L,
                                            int lane) {
    const double s = 1.0 / (double)L;
    bool b = false;
    for (int t = lane; t <= L / 2; t += 32) {
        const double2 hv = H[t];
        const double v0 = (t ? hv.x - hv.y : hv.x) * s;
        out[t] = v0;
        b |= fin_bad(v0);
        if (t) {
            const double v1 = (hv.x + hv.y) * s;
            out[L - t] = v1;
            b |= fin_bad(v1);
        }
    }
    __syncwarp();
    return b;
}

// rfft of the real series x (length L, in buffer xa) -> X[0 .. L/2]
// (complex, bins = L/2 + 1).  xb is scratch of the same capacity (>= 2L + 2
// doubles for odd L).  Returns the buffer holding X; the other is free.
// split == false (even L only): return the packed M-point transform Z itself
// (the caller splits the bin pairs it needs, see op_spectral).
template <bool BLUE = true, bool R16 = false, bool ODD = true>
__device__ __forceinline__ double2* rfft_any(double* xa, double* xb, int L, const FftGeo& g, const double2* tw,
                                            int lane, bool split = true) {
    double2* za = reinterpret_cast<double2*>(xa);
    double2* zb = reinterpret_cast<double2*>(xb);
    // odd L: complexify into xb and take the N = L transform; even L: view
    // the real series as N = L/2 complex points (one call site either way,
    // to keep the FFT's code emitted once)
    if (ODD && g.oddreal == 1) {
        oddreal_pack(xa, zb, L, g.radix[g.npass - 1], lane);
    } else if (!g.packed) {
        for (int n = lane; n < L; n += 32) zb[n] = make_double2(xa[n], 0.0);
        __syncwarp();
    }
    double2* s0 = g.packed ? za : zb;
    double2* d0 = g.packed ? zb : za;
    double2* Z = fft_any<BLUE, R16, false, ODD>(s0, d0, g, tw, L, lane);  // one call site: the FFT is emitted once
    if (!g.packed) {
        if (lane == 0) Z[0].y = 0.0;
        __syncwarp();
        return Z;
    }
    if (!split) return Z;
    const int M = L >> 1;
    double2* X = (Z == za) ? zb : za;
    // four bins per lane step, all loads first: independent latency chains
    for (int k0 = lane; k0 <= M; k0 += 128) {
        double2 zk[4], zc[4], wq[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int k = k0 + 32 * q <= M ? k0 + 32 * q : M;
            zk[q] = Z[k == M ? 0 : k];
            zc[q] = Z[k == 0 ? 0 : M - k];
            wq[q] = __ldg(&tw[k]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int k = k0 + 32 * q;
            double er = 0.5 * (zk[q].x + zc[q].x), ei = 0.5 * (zk[q].y - zc[q].y);
            double orr = 0.5 * (zk[q].y + zc[q].y), oi = -0.5 * (zk[q].x - zc[q].x);
            double2 o = cmul(make_double2(orr, oi), wq[q]);
            if (k <= M) X[k] = make_double2(er + o.x, ei + o.y);
        }
    }
    __syncwarp();
    if (lane == 0) {
        X[0].y = 0.0;
        X[M].y = 0.0;
    }
    __syncwarp();
    return X;
}

// irfft of X[0 .. L/2] (buffer X) to a real series of length L; `other` is
// free scratch.  Uses IFFT(Z) = conj(FFT(conj Z)).  Returns the buffer
// holding the series.  irfft ignores the imaginary part of the DC bin (and
// of the Nyquist bin for even L).
__device__ __forceinline__ bool fin_bad(double v) {  // exponent all ones: inf or nan
    return (__double2hiint(v) & 0x7ff00000) == 0x7ff00000;
}

// bad (optional): OR-ed with "some output is non-finite" in the final
// scaling loop, so callers need no separate pass over the row.
// folded == true (even L only): `other` already holds the folded M points
// (the conjugated inverse-FFT input); X is scratch.
template <bool BLUE = true, bool R16 = false, bool ODD = true>
__device__ __forceinline__ double* irfft_any(double2* X, double2* other, int L, const FftGeo& g, const double2* tw,
                                            int lane, bool* bad = nullptr, bool folded = false) {
    const int M = L >> 1;
    if (folded) {
    } else if (ODD && g.oddreal) {
        oddreal_fold(X, reinterpret_cast<double*>(other), L, lane);
        if (g.oddreal == 1) {
            oddreal_pack(reinterpret_cast<const double*>(other), X, L, g.radix[g.npass - 1], lane);
        } else {  // Bluestein on the half range of bins: the real series complexified
            const double* h = reinterpret_cast<const double*>(other);
            for (int n = lane; n < L; n += 32) X[n] = make_double2(h[n], 0.0);
        }
    } else if (!g.packed) {  // odd L: Hermitian completion, full transform, real part
        const int bins = L / 2 + 1;
        for (int k = lane; k < bins; k += 32) {
            double2 v = X[k];
            if (k == 0) v.y = 0.0;
            other[k] = make_double2(v.x, -v.y);
            if (k > 0) other[L - k] = v;
        }
    } else {  // even L: fold the half spectrum into M complex points (4 per lane step)
        for (int k0 = lane; k0 < M; k0 += 128) {
            double2 xk[4], xc[4], wq[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int k = k0 + 32 * q < M ? k0 + 32 * q : M - 1;
                xk[q] = X[k];
                xc[q] = X[M - k];
                wq[q] = __ldg(&tw[k]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int k = k0 + 32 * q;
                if (k == 0) { xk[q].y = 0.0; xc[q].y = 0.0; }
                xc[q].y = -xc[q].y;
                double er = 0.5 * (xk[q].x + xc[q].x), ei = 0.5 * (xk[q].y + xc[q].y);
                double dr = 0.5 * (xk[q].x - xc[q].x), di = 0.5 * (xk[q].y - xc[q].y);
                double2 w = wq[q];
                w.y = -w.y;
                double2 o = cmul(make_double2(dr, di), w);
                if (k < M) other[k] = make_double2(er - o.y, -(ei + o.x));
            }
        }
    }
    __syncwarp();
    bool fb = false;
    const bool odd = ODD && g.oddreal;
    double2* Z = fft_any<BLUE, R16, true, ODD>(odd ? X : other, odd ? other : X, g, tw, L, lane,
                                              &fb);  // one call site: the FFT is emitted once
    if (g.packed && is_fft_512(g, L)) {  // scaled and checked by the last pass
        if (bad) *bad |= fb;
        __syncwarp();
        return reinterpret_cast<double*>(Z);
    }
    if (odd) {
        double* out = reinterpret_cast<double*>(Z == X ? other : X);
        const bool b = oddreal_unfold(Z, out, L, lane);
        if (bad) *bad |= b;
        return out;
    }
    if (!g.packed) {
        double* out = reinterpret_cast<double*>(Z == X ? other : X);
        const double s = 1.0 / (double)L;
        bool b = false;
        for (int n = lane; n < L; n += 32) {
            const double v = Z[n].x * s;
            out[n] = v;
            b |= fin_bad(v);
        }
        if (bad) *bad |= b;
        __syncwarp();
        return out;
    }
    const double s = 1.0 / (double)M;
    bool b = false;
#pragma unroll 4
    for (int k = lane; k < M; k += 32) {
        double2 z = Z[k];
        const double2 v = make_double2(z.x * s, -(z.y * s));
        Z[k] = v;
        b |= fin_bad(v.x) | fin_bad(v.y);
    }
    if (bad) *bad |= b;
    __syncwarp();
    return reinterpret_cast<double*>(Z);
}


// ---------------------------------------------------------------- DCT
// Orthonormal DCT-II / DCT-III (scipy.fft.dct / idct, type 2, norm="ortho";
// reference freqtransform.py:91-98) of length N through one real FFT of
// length N (Makhoul): v[n] = x[2n], v[N-1-n] = x[2n+1] is real, so its
// spectrum V is Hermitian and the packed real transform (rfft_any: N/2
// complex points for even N) gives V[0 .. N/2]; V[k] = conj(V[N-k]) above.
//   S[k] = Re(e^{-i pi k / 2N} V[k]),  y[k] = g_k S[k],
//   g_0 = 1/sqrt(N), g_k = sqrt(2/N);
// inverse: V[k] = e^{+i pi k / 2N} (S[k] - i S[N-k]) (S[N] = 0) for
// k <= N/2, v = irfft(V).  dtw[k] = e^{-i pi k / 2N} (k < N); g / tw: the
// real-FFT plan and table of length N.  Buffers xa, xb hold the real-FFT
// capacity (N + 2 doubles for even N).  Returns the buffer with the result.
__device__ __forceinline__ double* dct2_any(double* xa, double* xb, int N, const FftGeo& g, const double2* tw,
                                           const double2* dtw, int lane) {
    for (int n = lane; n < N; n += 32) xb[n] = xa[(2 * n < N) ? 2 * n : 2 * (N - 1 - n) + 1];
    __syncwarp();
    double2* V = rfft_any<true, true>(xb, xa, N, g, tw, lane);
    double* y = (reinterpret_cast<double*>(V) == xa) ? xb : xa;
    const double g0 = 1.0 / sqrt((double)N), gk = sqrt(2.0 / (double)N);
    for (int k = lane; k < N; k += 32) {
        const double2 w = __ldg(&dtw[k]);
        double2 v = V[2 * k <= N ? k : N - k];
        v.y = 2 * k <= N ? v.y : -v.y;
        y[k] = (k == 0 ? g0 : gk) * (v.x * w.x - v.y * w.y);
    }
    __syncwarp();
    return y;
}

__device__ __forceinline__ double* dct3_any(double* ya, double* yb, int N, const FftGeo& g, const double2* tw,
                                           const double2* dtw, int lane) {
    double2* V = reinterpret_cast<double2*>(yb);
    const double i0 = sqrt((double)N), ik = sqrt((double)N / 2.0);
    for (int k = lane; 2 * k <= N; k += 32) {
        const double sk = ya[k] * (k == 0 ? i0 : ik);
        const double snk = (k == 0) ? 0.0 : ya[N - k] * ik;
        double2 w = __ldg(&dtw[k]);
        w.y = -w.y;  // e^{+i pi k / 2N}
        V[k] = cmul(make_double2(sk, -snk), w);
    }
    __syncwarp();
    double* v = irfft_any<true, true>(V, reinterpret_cast<double2*>(ya), N, g, tw, lane);
    double* x = (v == ya) ? yb : ya;
    for (int n = lane; n < N; n += 32) x[(2 * n < N) ? 2 * n : 2 * (N - 1 - n) + 1] = v[n];
    __syncwarp();
    return x;
}

}  // namespace sa
