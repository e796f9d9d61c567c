// sa_ops.cuh -- the augmentation operators, one warp per series, series in smem.
//
// Each op transforms `cur` (length L) and may use `oth` as scratch or as the
// output buffer (then it swaps the two).  All draws come from the stage's
// WStream in exactly the reference's order (gate first, consumed by the
// pre-pass in the kernel).  FP expressions follow the reference's evaluation
// order; the TU is compiled with -fmad=false so nothing is contracted.
#pragma once
#include <math.h>
#include <stdint.h>

#include "../../include/seriesaug_b200.h"
#include "sa_fft.cuh"
#include "sa_rng.cuh"

#define SA_MAX_AUX 512

namespace sa {

struct DevStage {
    int32_t op, index;
    int32_t len_in, len_out;
    int32_t post_repeat, aux_off;
    int32_t aux_len, pad;
    double prob;
    double f[4];
    int64_t i[4];
    const double2* tw;  // exp(-2 pi i k / len_in), k < len_in (spectral ops)
    FftGeo fft;         // transform plan for len_in (spectral ops)
};

struct ChainParams {
    int32_t ns, repeat_r;
    int32_t len_in, len_out;
    int32_t lcap, small_words, iscr_words, bulk_in;
    int32_t sync_every, key_bits;  // sync_every != 0: barriers on; fire-pattern key width
    uint64_t sync_mask;            // bit j: CTA barrier before stage j
    uint64_t uni_mask;             // gates compared across the CTA's rows; all equal -> no in-row barriers
    const int32_t* order;          // row schedule (nullptr: identity)
    int8_t key_stage[24];          // stages whose gates form the key, most expensive first
    uint64_t seed;
    int64_t offset;
    int64_t rows_out;
    const double* in;
    double* out;
    uint32_t* flags;
    double* gbuf;                  // non-null: row buffers in global memory (series too long for smem)
    double aux[SA_MAX_AUX];
    DevStage st[SA_MAX_STAGES];
};

struct Warp {
    int lane;
    const ZigEntry* zig;  // ziggurat fast-path table (smem copy in the chain kernel)
    uint64_t* win;
    double* small;
    int32_t* iscr;
    int lcap;
};

// ---------------------------------------------------------------- numerics
// np.linspace(start, stop, num)[k], endpoint=True (numpy function_base).
__device__ __forceinline__ double linspace_at(double start, double stop, int64_t num, int64_t k) {
    if (num > 1 && k == num - 1) return stop;
    int64_t div = num - 1;
    double delta = stop - start;
    double y = (double)k;
    if (div > 0) {
        double step = delta / (double)div;
        if (step == 0.0) y = (y / (double)div) * delta;
        else y = y * step;
    } else {
        y = y * delta;
    }
    return y + start;
}

// np.linspace(start, stop, num) with its step hoisted out of element loops:
// element k is (double)k * step + start (step != 0) or ((double)k / div) * delta
// + start (step == 0), the last element pinned to stop.
struct Linspace {
    double start, stop, step, delta;
    int64_t num, div;
    bool zero;
    __device__ __forceinline__ Linspace(double a, double b, int64_t n) : start(a), stop(b), num(n), div(n - 1) {
        delta = b - a;
        step = div > 0 ? delta / (double)div : 0.0;
        zero = div > 0 && step == 0.0;
    }
    // the common case (num > 1, step != 0): k * step + start, last = stop
    __device__ __forceinline__ bool fast() const { return div > 0 && !zero; }
    __device__ __forceinline__ double at_fast(int k) const {
        const double y = (double)k * step + start;
        return k == num - 1 ? stop : y;
    }
    __device__ __forceinline__ double at(int64_t k) const {
        if (num > 1 && k == num - 1) return stop;
        double y = (double)k;
        if (div > 0) y = zero ? (y / (double)div) * delta : y * step;
        else y = y * delta;
        return y + start;
    }
};

// np.interp on a linspace table xp with precomputed per-interval slopes
// (numpy precomputes exactly these slopes when len(xp) <= len(x)).  The
// bracketing interval comes from the O(1) guess hint = (int)(x / step),
// which on a linspace table is off by at most one (both sides round within
// an ulp), so one compare each way yields numpy's "largest j with
// xp[j] <= x"; no search loop, so unrolled calls interleave.  Every caller
// (Drift anchors, TimeWarp / WindowWarp knots) passes a linspace table.
__device__ __forceinline__ double interp_slopes(double x, const double* __restrict__ xp, const double* __restrict__ fp,
                                                const double* __restrict__ sl, int n, int hint) {
    int j = hint < 0 ? 0 : (hint > n - 2 ? n - 2 : hint);
    j = (xp[j + 1] <= x && j < n - 2) ? j + 1 : j;
    j = (xp[j] > x && j > 0) ? j - 1 : j;
    const double xj = xp[j], fj = fp[j];
    double r = sl[j] * (x - xj) + fj;
    r = (xj == x) ? fj : r;
    r = (x >= xp[n - 1]) ? fp[n - 1] : r;
    r = (x < xp[0]) ? fp[0] : r;
    return r;
}

// np.interp(t, xp, fp) for every integer t in [0, L), xp non-decreasing,
// with numpy's precomputed slopes sl: segment by segment, so the bracketing
// interval ("largest j with xp[j] <= t") is warp-uniform and held in
// registers -- no per-element search or table loads.  f(t, value) is called
// exactly once per t, by one lane.  Same arithmetic as interp_slopes.
template <class F>
__device__ __forceinline__ void interp_arange(const double* __restrict__ xp, const double* __restrict__ fp,
                                              const double* __restrict__ sl, int n, int L, int lane, F&& f) {
    int t = (int)ceil(xp[0]);  // t < xp[0]: fp[0]
    t = t < 0 ? 0 : (t > L ? L : t);
    for (int u = lane; u < t; u += 32) f(u, fp[0]);
    for (int j = 0; j < n - 1 && t < L; ++j) {
        const double xj = xp[j], fj = fp[j], sj = sl[j];
        int te = (int)ceil(xp[j + 1]);  // first t of the next segment
        te = te > L ? L : te;
#pragma unroll 4
        for (int u = t + lane; u < te; u += 32) {
            const double x = (double)u;
            double r = sj * (x - xj) + fj;
            r = (xj == x) ? fj : r;
            f(u, r);
        }
        t = te > t ? te : t;
    }
    const double fl = fp[n - 1];  // t >= xp[n-1]
    for (int u = t + lane; u < L; u += 32) f(u, fl);
}

// np.interp(x, xp, fp) with xp increasing (binary search, exact-hit rule).
__device__ __forceinline__ double interp1(double x, const double* xp, const double* fp, int n) {
    if (x > xp[n - 1]) return fp[n - 1];
    if (x < xp[0]) return fp[0];
    int lo = 0, hi = n;
    while (hi - lo > 1) {
        int mid = lo + ((hi - lo) >> 1);
        if (x >= xp[mid]) lo = mid;
        else hi = mid;
    }
    int j = lo;
    if (j == n - 1) return fp[j];
    if (xp[j] == x) return fp[j];
    double slope = (fp[j + 1] - fp[j]) / (xp[j + 1] - xp[j]);
    double r = slope * (x - xp[j]) + fp[j];
    if (isnan(r)) {
        r = slope * (x - xp[j + 1]) + fp[j + 1];
        if (isnan(r) && fp[j] == fp[j + 1]) r = fp[j];
    }
    return r;
}

__device__ __forceinline__ bool nonfinite(double v) {
    return (__double2hiint(v) & 0x7ff00000) == 0x7ff00000;
}

// Per-lane finiteness accumulator for the values a stage writes (the
// reference re-validates every stage's output Batch, core.py:259 -> :104):
// s + v * 0 is NaN iff some v was inf / NaN and stays exactly 0 otherwise, so
// ONE DFMA per checked value (on the FP64 pipe, which the chain leaves mostly
// idle) replaces the exponent test's LOP3 + ISETP + SEL + OR.
struct Finite {
    double s = 0.0;
    __device__ __forceinline__ void chk(double v) { s = fma(v, 0.0, s); }
    __device__ __forceinline__ void merge(bool b) {
        if (b) s = __longlong_as_double(0x7ff8000000000000ll);
    }
    __device__ __forceinline__ bool any() const { return s != s; }
};

// np.interp(x, arange(n), fp) for n >= 2, branch-free.  The reference's NaN
// fallback (numpy arr_interp) can only trigger for non-finite data, which the
// kernel rejects (SA_FLAG_NONFINITE), so it is not reproduced here.
__device__ __forceinline__ double interp_grid_fast(double x, const double* __restrict__ fp, int n) {
    const double fl = floor(x);
    int j = (int)fl;
    j = j < 0 ? 0 : (j > n - 2 ? n - 2 : j);
    const double a = fp[j], b = fp[j + 1];
    double r = (b - a) * (x - fl) + a;  // (x - xp[j]) with xp[j] = j = fl in range
    r = (x == fl) ? a : r;              // exact hit: fp[j]
    r = (x >= (double)(n - 1)) ? fp[n - 1] : r;
    r = (x < 0.0) ? fp[0] : r;
    return r;
}

// np.interp(x, arange(n), fp).
__device__ __forceinline__ double interp_grid(double x, const double* fp, int n) {
    if (x > (double)(n - 1)) return fp[n - 1];
    if (x < 0.0) return fp[0];
    int j = (int)floor(x);
    if (j >= n - 1) return fp[n - 1];
    if ((double)j == x) return fp[j];
    // xp = arange(n): (j+1) - j == 1.0 exactly and d / 1.0 == d, so the
    // reference's slope is the plain difference (no division needed)
    double slope = fp[j + 1] - fp[j];
    double r = slope * (x - (double)j) + fp[j];
    if (isnan(r)) {
        r = slope * (x - (double)(j + 1)) + fp[j + 1];
        if (isnan(r) && fp[j] == fp[j + 1]) r = fp[j];
    }
    return r;
}

// numpy pairwise summation (np.add.reduce on contiguous float64,
// pairwise_sum_DOUBLE): n < 8 -> sequential; n <= 128 -> a leaf with 8
// strided accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then
// the n % 8 tail added in order; n > 128 -> split at n2 = n/2 - (n/2) % 8.
// Leaves are summed in parallel (8 lanes per leaf, one accumulator each) and
// combined in the recursion's order by an iterative post-order walk.
struct PwFrame {
    int n, stage;
    double left;
};

__device__ __forceinline__ int pw_split(int n) {
    int n2 = n / 2;
    return n2 - n2 % 8;
}

// Leaves of the recursion over [0, n) in left-to-right order -> (start, len).
__device__ __noinline__ int pairwise_leaf_list(int n, int2* leaves) {
    int lo_stack[32], n_stack[32];
    int sp = 0, cnt = 0;
    lo_stack[0] = 0;
    n_stack[0] = n;
    while (sp >= 0) {
        const int lo = lo_stack[sp], m = n_stack[sp];
        --sp;
        if (m <= 128) {
            leaves[cnt++] = make_int2(lo, m);
        } else {
            const int n2 = pw_split(m);
            ++sp; lo_stack[sp] = lo + n2; n_stack[sp] = m - n2;  // right, popped second
            ++sp; lo_stack[sp] = lo; n_stack[sp] = n2;           // left, popped first
        }
    }
    return cnt;
}

__device__ __noinline__ double pairwise_combine(int n, const double* leafsum) {
    PwFrame st[32];
    int sp = 0, leaf = 0;
    st[0].n = n; st[0].stage = 0; st[0].left = 0.0;
    for (;;) {
        PwFrame& f = st[sp];
        if (f.n <= 128) {
            double v = leafsum[leaf++];
            for (;;) {
                if (sp == 0) return v;
                --sp;
                PwFrame& par = st[sp];
                if (par.stage == 1) {  // left child done: descend right
                    par.left = v;
                    par.stage = 2;
                    ++sp;
                    st[sp].n = par.n - pw_split(par.n); st[sp].stage = 0; st[sp].left = 0.0;
                    break;
                }
                v = par.left + v;  // right child done
            }
        } else {
            f.stage = 1;
            const int n2 = pw_split(f.n);
            ++sp;
            st[sp].n = n2; st[sp].stage = 0; st[sp].left = 0.0;
        }
    }
}

// n a power of two >= 128: the recursion's leaves are the 128-blocks and
// its combine tree is perfect, so no leaf list / post-order walk is needed.
// 8 lanes per leaf (numpy's 8 strided accumulators), a shfl_xor butterfly
// for ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), two shfl_down levels join the
// 4 leaves of a pass, and a perfect tree over the passes' sums (scratch).
template <class F>
__device__ __forceinline__ double pairwise_warp_pow2(int n, F f, double* scratch, int lane) {
    const int nl = n >> 7;
    const int passes = (nl + 3) >> 2;
    const int g = lane >> 3, q = lane & 7;
    double res = 0.0;
    for (int ps = 0; ps < passes; ++ps) {
        const int l = 4 * ps + g;
        double acc = 0.0;
        if (l < nl) {
            const int base = 128 * l + q;
            acc = f(base);
#pragma unroll
            for (int k = 1; k < 16; ++k) acc += f(base + 8 * k);
        }
        acc = acc + __shfl_xor_sync(SA_FULL, acc, 1);
        acc = acc + __shfl_xor_sync(SA_FULL, acc, 2);
        acc = acc + __shfl_xor_sync(SA_FULL, acc, 4);
        double o = __shfl_down_sync(SA_FULL, acc, 8);
        if (nl >= 2) acc = acc + o;
        o = __shfl_down_sync(SA_FULL, acc, 16);
        if (nl >= 4) acc = acc + o;
        if (passes == 1) res = acc;
        else if (lane == 0) scratch[ps] = acc;
    }
    if (passes > 1) {
        __syncwarp();
        for (int h = 1; h < passes; h *= 2) {
            for (int i = lane; 2 * h * i < passes; i += 32) scratch[2 * h * i] = scratch[2 * h * i] + scratch[2 * h * i + h];
            __syncwarp();
        }
        res = scratch[0];
        __syncwarp();
    }
    return __shfl_sync(SA_FULL, res, 0);
}

// Pairwise sum of f(t), t < n.  scratch: >= 2 * (n / 64 + 2) doubles.
template <class F>
__device__ double pairwise_warp(int n, F f, double* scratch, int lane) {
    if (n >= 128 && (n & (n - 1)) == 0) return pairwise_warp_pow2(n, f, scratch, lane);
    if (n < 8) {
        double r = 0.0;
        for (int k = 0; k < n; ++k) r += f(k);
        return r;
    }
    int2* leaves = reinterpret_cast<int2*>(scratch);
    const int nl_max = n / 64 + 2;
    double* leafsum = scratch + nl_max;
    int nl;
    if (lane == 0) nl = pairwise_leaf_list(n, leaves);
    nl = __shfl_sync(SA_FULL, nl, 0);
    __syncwarp();
    const int g = lane >> 3, q = lane & 7;
    for (int l0 = 0; l0 < nl; l0 += 4) {
        const int l = l0 + g;
        double acc = 0.0, res = 0.0;
        int2 lf = make_int2(0, 0);
        if (l < nl) {
            lf = leaves[l];
            const int full = lf.y - lf.y % 8;
            acc = f(lf.x + q);
            for (int k = 8 + q; k < full; k += 8) acc += f(lf.x + k);
        }
        // gather the group's 8 accumulators to its first lane, numpy's order
        double r[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = __shfl_sync(SA_FULL, acc, (lane & ~7) + u);
        if (q == 0 && l < nl) {
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
            for (int k = lf.y - lf.y % 8; k < lf.y; ++k) res += f(lf.x + k);
            leafsum[l] = res;
        }
    }
    __syncwarp();
    double total = pairwise_combine(n, leafsum);
    __syncwarp();
    return total;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        double u = __shfl_xor_sync(SA_FULL, v, o);
        v = (u < v) ? u : v;
    }
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        double u = __shfl_xor_sync(SA_FULL, v, o);
        v = (u > v || u != u) ? u : v;
    }
    return v;
}

__device__ __forceinline__ void swapbuf(double*& a, double*& b) {
    double* t = a;
    a = b;
    b = t;
}

// ---------------------------------------------------------------- operators
// All return true when the op did arithmetic (so the kernel re-checks
// finiteness), false for pure index moves / no-ops.

// basic.py:41-44 Jitter, basic.py:356-359 InjectNoise(gaussian):
// y = x + (0.0 + sigma * z)
__device__ __forceinline__ bool op_gauss(const DevStage& st, WStream& s, double*& cur, double*& oth, int& L, Warp& w, Finite& bad) {
    const double sigma = st.f[0];
    if (sigma == 0.0) return false;
    double* x = cur;
    normals(s, w.lane, L, w.zig, [&](int k, double z) {
        const double v = x[k] + (0.0 + sigma * z);
        x[k] = v;
        bad.chk(v);
    });
    __syncwarp();
    return false;
}

// basic.py:58-60 Scale: s = 1.0 + sigma_factor * z; y = x * s
__device__ __forceinline__ bool op_scale(const DevStage& st, WStream& s, double*& cur, double*& oth, int& L, Warp& w, Finite& bad) {
    double f = 1.0 + st.f[0] * std_normal(s, w.lane);
    for (int t = w.lane; t < L; t += 32) {
        const double v = cur[t] * f;
        cur[t] = v;
        bad.chk(v);
    }
    __syncwarp();
    return false;
}

// basic.py:70-71 Rotate: -x
__device__ __forceinline__ bool op_rotate(double*& cur, int L, Warp& w) {
    for (int t = w.lane; t < L; t += 32) cur[t] = -cur[t];
    __syncwarp();
    return false;
}

// basic.py:95-104 PermuteSegments
__device__ __forceinline__ bool op_permute(const DevStage& st, WStream& s, double*& cur, double*& oth, int& L, Warp& w) {
    const int n = (int)st.i[0];
    if (n == 1) return false;
    int32_t* order = w.iscr;
    for (int k = w.lane; k < n; k += 32) order[k] = k;
    __syncwarp();
    for (int i = n - 1; i > 0; --i) {  // Generator.permutation: Fisher-Yates
        int j = (int)interval(s, w.lane, (uint32_t)i);
        if (w.lane == 0) {
            int32_t t = order[i];
            order[i] = order[j];
            order[j] = t;
        }
        __syncwarp();
    }
    const int base = L / n, extra = L % n;
    int o = 0;
    for (int q = 0; q < n; ++q) {
        int k = order[q];
        int off = k * base + (k < extra ? k : extra);
        int sz = base + (k < extra ? 1 : 0);
        for (int u = w.lane; u < sz; u += 32) oth[o + u] = cur[off + u];
        o += sz;
    }
    __syncwarp();
    swapbuf(cur, oth);
    return false;
}

// basic.py:133-135 Crop: start = integers(0, L - size + 1)
__device__ __forceinline__ bool op_crop(const DevStage& st, WStream& s, double*& cur, double*& oth, int& L, Warp& w) {
    const int size = (int)st.i[0];
    const int start = (int)bounded(s, w.lane, (uint32_t)(L - size));
    for (int t = w.lane; t < size; t += 32) oth[t] = cur[start + t];
    __syncwarp();
    swapbuf(cur, oth);
    L = size;
    return false;
}

// basic.py:145-146 Reverse
__device__ __forceinline__ bool op_reverse(double*& cur, double*& oth, int L, Warp& w) {
    for (int t = w.lane; t < L; t += 32) oth[t] = cur[L - 1 - t];
    __syncwarp();
    swapbuf(cur, oth);
    return false;
}

// basic.py:174-177 Resize: interp(linspace(0, L-1, T), arange(L), x)
__device__ __forceinline__ bool op_resize(const DevStage& st, double*& cur, double*& oth, int& L, Warp& w, Finite& bad) {
    const int T = (int)st.i[0];
    if (T == L) return false;
    const Linspace ls(0.0, (double)L - 1.0, T);
    if (ls.fast()) {
#pragma unroll 4
        for (int t = w.lane; t < T; t += 32) {
            const double v = interp_grid_fast(ls.at_fast(t), cur, L);
            oth[t] = v;
            bad.chk(v);
        }
    } else {
        for (int t = w.lane; t < T; t += 32) {
            const double v = interp_grid(ls.at(t), cur, L);
            oth[t] = v;
            bad.chk(v);
        }
    }
    __syncwarp();
    swapbuf(cur, oth);
    L = T;
    return false;
}

// basic.py:196-207 Quantize / snap_to_levels
__device__ __forceinline__ bool op_quantize(const DevStage& st, double*& cur, int L, Warp& w, Finite& bad) {
    double lo = cur[0], hi = cur[0];
    for (int t = w.lane; t < L; t += 32) {
        double v = cur[t];
        lo = (v < lo) ? v : lo;
        hi = (v > hi) ? v : hi;
    }
    lo = warp_min(lo);
    hi = warp_max(hi);
    if (hi == lo) return false;
    const double step = (hi - lo) / (double)(st.i[0] - 1);
    const double top = (double)(st.i[0] - 1);
    for (int t = w.lane; t < L; t += 32) {
        double idx = ceil((cur[t] - lo) / step - 0.5);
        idx = (idx < 0.0) ? 0.0 : idx;  // np.clip keeps -0.0 (x < 0 is false)
        idx = (idx > top) ? top : idx;
        const double v = lo + idx * step;
        cur[t] = v;
        bad.chk(v);
    }
    __syncwarp();
    return false;
}

// basic.py:227-241 Drift: anchors ~ N(0,1)^n at linspace(0, L-1, n),
// curve = interp(arange(L), positions, anchors) - curve[0], scaled so its peak
// magnitude is max_drift.
__device__ __forceinline__ bool op_drift(const DevStage& st, WStream& s, double*& cur, double*& oth, int L, Warp& w, Finite& bad) {
    const double md = st.f[0];
    if (md == 0.0) return false;
    const int np_ = (int)st.i[0];
    double* anchors = w.small;
    double* pos = w.small + np_;
    double* sl = w.small + 2 * np_;
    for (int k = 0; k < np_; ++k) {
        double a = 0.0 + 1.0 * std_normal(s, w.lane);
        if (w.lane == 0) anchors[k] = a;
    }
    const Linspace ls(0.0, (double)L - 1.0, np_);
    for (int k = w.lane; k < np_; k += 32) pos[k] = ls.at(k);
    __syncwarp();
    for (int k = w.lane; k < np_ - 1; k += 32) sl[k] = (anchors[k + 1] - anchors[k]) / (pos[k + 1] - pos[k]);
    __syncwarp();
    const double c0 = interp_slopes(0.0, pos, anchors, sl, np_, 0);
    double* curve = oth;  // pass 1: curve - c0 and its peak
    double peak = 0.0;
    interp_arange(pos, anchors, sl, np_, L, w.lane, [&](int t, double v) {
        const double c = v - c0;
        curve[t] = c;
        const double a = fabs(c);
        peak = (a > peak || a != a) ? a : peak;
    });
    peak = warp_max(peak);
    if (peak == 0.0) return false;
#pragma unroll 4
    for (int t = w.lane; t < L; t += 32) {
        const double v = cur[t] + (curve[t] / peak) * md;
        cur[t] = v;
        bad.chk(v);
    }
    __syncwarp();
    return false;
}

// basic.py:352-355 InjectNoise(uniform): x + uniform(-hw, hw)
__device__ __forceinline__ bool op_uniform(const DevStage& st, WStream& s, double*& cur, int L, Warp& w, Finite& bad) {
    const double hw = st.f[0];
    if (hw == 0.0) return false;
    const double lo = -hw, range = hw - lo;
    double* x = cur;
    doubles(s, w.lane, L, [&](int k, double u) {
        const double v = x[k] + (lo + range * u);
        x[k] = v;
        bad.chk(v);
    });
    __syncwarp();
    return false;
}

// Generator.choice(L, k, replace=False) into idx[0..k) (int32 scratch).
__device__ __noinline__ void choice_noreplace(WStream& s, int lane, int pop, int k, int32_t* iscr, int32_t* idx) {
    if (pop > 10000 && k > pop / 50) {  // tail shuffle of arange(pop)
        int32_t* a = iscr;
        for (int t = lane; t < pop; t += 32) a[t] = t;
        __syncwarp();
        int first = pop - k > 1 ? pop - k : 1;
        for (int i = pop - 1; i >= first; --i) {
            int j = (int)bounded(s, lane, (uint32_t)i);
            if (lane == 0) {
                int32_t t = a[i];
                a[i] = a[j];
                a[j] = t;
            }
            __syncwarp();
        }
        for (int t = lane; t < k; t += 32) idx[t] = a[pop - k + t];
        __syncwarp();
        return;
    }
    uint32_t mask = (uint32_t)(1.2 * (double)k);
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4; mask |= mask >> 8; mask |= mask >> 16;
    uint32_t* hs = reinterpret_cast<uint32_t*>(iscr);
    for (uint32_t t = lane; t <= mask; t += 32) hs[t] = 0xffffffffu;
    __syncwarp();
    for (int j = pop - k; j < pop; ++j) {
        uint32_t val = bounded(s, lane, (uint32_t)j);
        uint32_t loc = val & mask;
        while (hs[loc] != 0xffffffffu && hs[loc] != val) loc = (loc + 1) & mask;
        int32_t pick;
        if (hs[loc] == 0xffffffffu) {
            pick = (int32_t)val;
        } else {
            loc = (uint32_t)j & mask;
            while (hs[loc] != 0xffffffffu) loc = (loc + 1) & mask;
            val = (uint32_t)j;
            pick = j;
        }
        __syncwarp();
        if (lane == 0) {
            hs[loc] = val;
            idx[j - pop + k] = pick;
        }
        __syncwarp();
    }
    for (int i = k - 1; i > 0; --i) {
        int j = (int)bounded(s, lane, (uint32_t)i);
        if (lane == 0) {
            int32_t t = idx[i];
            idx[i] = idx[j];
            idx[j] = t;
        }
        __syncwarp();
    }
}

// basic.py:360-370 InjectNoise(spike)
__device__ __forceinline__ bool op_spike(const DevStage& st, WStream& s, double*& cur, double*& oth, int L, Warp& w, Finite& bad) {
    const int cnt = (int)st.i[0];
    const double mag = st.f[0];
    if (cnt == 0 || mag == 0.0) return false;
    const double* x = cur;
    double mean = pairwise_warp(L, [&](int t) { return x[t]; }, w.small, w.lane) / (double)L;
    double var = pairwise_warp(
                     L, [&](int t) { double d = x[t] - mean; return d * d; }, w.small, w.lane) /
                 (double)L;
    double scale = sqrt(var);
    if (scale == 0.0) scale = 1.0;
    // hash set / tail array first, picks after it (host sizes lcap for it)
    uint32_t mask = (uint32_t)(1.2 * (double)cnt);
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4; mask |= mask >> 8; mask |= mask >> 16;
    int scr = (L > 10000 && cnt > L / 50) ? L : (int)mask + 1;
    int32_t* scratch = reinterpret_cast<int32_t*>(oth);  // free during this in-place op
    int32_t* idx = scratch + scr;
    WStream t = s;  // by-address copy for the out-of-line helper; s stays in registers
    choice_noreplace(t, w.lane, L, cnt, scratch, idx);
    s = t;
    for (int q = 0; q < cnt; ++q) {
        double sign = (double)((int64_t)bounded(s, w.lane, 1u) * 2 - 1);
        if (w.lane == 0) {
            int p = idx[q];
            const double v = cur[p] + (sign * mag) * scale;
            cur[p] = v;
            bad.chk(v);
        }
    }
    __syncwarp();
    return false;
}

// basic.py:371-375 InjectNoise(slope_trend)
__device__ __forceinline__ bool op_slope(const DevStage& st, WStream& s, double*& cur, int L, Warp& w, Finite& bad) {
    const double mo = st.f[0];
    if (mo == 0.0) return false;
    const double sign = next_double(s, w.lane) < 0.5 ? 1.0 : -1.0;
    const double stop = sign * mo;
    const Linspace ls(0.0, stop, L);
    if (ls.fast()) {
#pragma unroll 4
        for (int t = w.lane; t < L; t += 32) {
            const double v = cur[t] + ls.at_fast(t);
            cur[t] = v;
            bad.chk(v);
        }
    } else {
        for (int t = w.lane; t < L; t += 32) {
            const double v = cur[t] + ls.at(t);
            cur[t] = v;
            bad.chk(v);
        }
    }
    __syncwarp();
    return false;
}

// warp.py:25-47 warp_positions: builds knots (small[0..n)) and warped
// (small[n..2n)); returns false if the map is not strictly increasing.
__device__ __noinline__ bool warp_knots(int len, int nk, double intensity, WStream& s, Warp w) {
    const double span = (double)len - 1.0;
    double* knots = w.small;
    double* warped = w.small + nk;
    double* tmp = w.small + 2 * nk;
    const double spacing = span / (double)(nk - 1);
    const Linspace ls(0.0, span, nk);
    for (int k = w.lane; k < nk; k += 32) knots[k] = ls.at(k);
    __syncwarp();
    const int ni = nk - 2;
    for (int k = 0; k < ni; ++k) {
        double v = knots[k + 1] + (0.0 + (intensity * spacing) * std_normal(s, w.lane));
        if (w.lane == 0) tmp[k] = v;
    }
    __syncwarp();
    if (w.lane == 0) {
        for (int a = 1; a < ni; ++a) {  // np.sort (values)
            double v = tmp[a];
            int b = a - 1;
            while (b >= 0 && tmp[b] > v) {
                tmp[b + 1] = tmp[b];
                --b;
            }
            tmp[b + 1] = v;
        }
        double prev = 0.0, acc = 0.0;
        warped[0] = 0.0;
        for (int k = 1; k < nk; ++k) {
            double cur = (k == nk - 1) ? span : tmp[k - 1];
            if (k < nk - 1) {  // np.clip(sorted, 0, span)
                if (cur < 0.0) cur = 0.0;
                if (cur > span) cur = span;
            }
            double g = cur - prev;
            if (!(g >= 1e-6)) g = (g != g) ? g : 1e-6;
            prev = cur;
            acc = acc + g;
            warped[k] = acc;
        }
        const double f = span / warped[nk - 1];
        for (int k = 0; k < nk; ++k) warped[k] = warped[k] * f;
        warped[nk - 1] = span;
    }
    __syncwarp();
    double* sl = w.small + 2 * nk;  // interp slopes of the map (tmp no longer needed)
    for (int k = w.lane; k < nk - 1; k += 32) sl[k] = (warped[k + 1] - warped[k]) / (knots[k + 1] - knots[k]);
    __syncwarp();
    bool ok = true;
    for (int k = 1; k < nk; ++k) ok = ok && !(warped[k] - warped[k - 1] <= 0);
    return ok;
}

// warp.py:73-76 TimeWarp
__device__ __forceinline__ bool op_time_warp(const DevStage& st, WStream& s, double*& cur, double*& oth, int L, Warp& w,
                             uint32_t& flags, Finite& bad) {
    if (st.f[0] == 0.0) return false;
    const int nk = (int)st.i[0];
    WStream t = s;
    const bool ok = warp_knots(L, nk, st.f[0], t, w);
    s = t;
    if (!ok) {
        flags |= SA_FLAG_WARP_MONOTONE;
        return false;
    }
    const double* knots = w.small;
    const double* warped = w.small + nk;
    const double* sl = w.small + 2 * nk;
    interp_arange(knots, warped, sl, nk, L, w.lane, [&](int t, double pos) {
        const double v = interp_grid_fast(pos, cur, L);
        oth[t] = v;
        bad.chk(v);
    });
    __syncwarp();
    swapbuf(cur, oth);
    return false;
}

// warp.py:108-118 WindowWarp
__device__ __forceinline__ bool op_window_warp(const DevStage& st, WStream& s, double*& cur, double*& oth, int L, Warp& w,
                               uint32_t& flags, Finite& bad) {
    if (st.f[0] == 0.0) return false;
    const int wsz = (int)st.i[0];
    const int nk = (int)st.i[1];
    const int start = (wsz == L) ? 0 : (int)bounded(s, w.lane, (uint32_t)(L - wsz));
    WStream t = s;
    const bool ok = warp_knots(wsz, nk, st.f[0], t, w);
    s = t;
    if (!ok) {
        flags |= SA_FLAG_WARP_MONOTONE;
        return false;
    }
    const double* knots = w.small;
    const double* warped = w.small + nk;
    const double* sl = w.small + 2 * nk;
    const double* win = cur + start;
    double* wout = oth + start;
    interp_arange(knots, warped, sl, nk, wsz, w.lane, [&](int u, double pos) {
        const double v = interp_grid_fast(pos, win, wsz);
        wout[u] = v;
        bad.chk(v);
    });
    // the complement is untouched (warp.py:108-118)
#pragma unroll 4
    for (int t = w.lane; t < L; t += 32)
        if (t < start || t >= start + wsz) oth[t] = cur[t];
    __syncwarp();
    swapbuf(cur, oth);
    return false;
}

// BASELINE M2 Dropout
__device__ __forceinline__ bool op_dropout(const DevStage& st, WStream& s, double*& cur, int L, Warp& w) {
    const double rate = st.f[0], fill = st.f[1];
    if (rate == 0.0) return false;
    double* x = cur;
    doubles(s, w.lane, L, [&](int k, double u) {
        if (u < rate) x[k] = fill;
    });
    __syncwarp();
    return false;
}

// BASELINE M3 Pool
__device__ __forceinline__ bool op_pool(const DevStage& st, double*& cur, int L, Warp& w, Finite& bad) {
    const int P = (int)st.i[0];
    if (P == 1) return false;
    const int red = (int)st.i[1];
    const int nb = (L + P - 1) / P;
    for (int b = w.lane; b < nb; b += 32) {
        int b0 = b * P, b1 = b0 + P < L ? b0 + P : L;
        double v;
        if (red == 0) {
            double acc = 0.0;
            for (int u = b0; u < b1; ++u) acc = acc + cur[u];
            v = acc / (double)(b1 - b0);
        } else if (red == 1) {
            v = cur[b0];
            for (int u = b0 + 1; u < b1; ++u) v = (cur[u] > v) ? cur[u] : v;
        } else {
            v = cur[b0];
            for (int u = b0 + 1; u < b1; ++u) v = (cur[u] < v) ? cur[u] : v;
        }
        for (int u = b0; u < b1; ++u) cur[u] = v;
        bad.chk(v);
    }
    __syncwarp();
    return false;
}

// BASELINE M4 Convolve (taps in params.aux).  Each lane computes four
// outputs (t + 32q) as independent chains; chunks whose taps stay inside
// the series skip the edge clamp.  Per output the taps are summed in order
// k = 0..S-1 exactly as before.
// Seven taps (the configs' size): lane pairs.  Each lane computes outputs
// t, t + 1 (t even) from five aligned 16-byte loads of x[t-4 .. t+5] (2.5
// loads per output instead of 7), four pairs per lane per step (eight
// independent accumulation chains); the <= 4 + 5 edge outputs whose taps
// reach past the series take the clamped path.
__device__ __forceinline__ void convolve7(const double* __restrict__ taps, const double* cur, double* oth, int L,
                                          Warp& w, Finite& bad) {
    double c[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) c[k] = taps[k];
    const int tmax = L - 6;  // last interior pair start: t + 5 <= L - 1
    const double2* c2 = reinterpret_cast<const double2*>(cur);
    for (int t0 = 4; t0 <= tmax; t0 += 256) {
        double acc[8];
        double2 v[4][5];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int t = t0 + 2 * w.lane + 64 * q;
            const int tl = t <= tmax ? t : 4;  // idle lanes read a valid pair
#pragma unroll
            for (int m = 0; m < 5; ++m) v[q][m] = c2[(tl - 4) / 2 + m];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            // x[t - 4 + i] for i = 0..9
            const double x[10] = {v[q][0].x, v[q][0].y, v[q][1].x, v[q][1].y, v[q][2].x,
                                  v[q][2].y, v[q][3].x, v[q][3].y, v[q][4].x, v[q][4].y};
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int k = 0; k < 7; ++k) {
                a0 = a0 + c[k] * x[1 + k];  // x[t + k - 3]
                a1 = a1 + c[k] * x[2 + k];  // x[t + 1 + k - 3]
            }
            acc[2 * q] = a0;
            acc[2 * q + 1] = a1;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int t = t0 + 2 * w.lane + 64 * q;
            if (t <= tmax) {
                reinterpret_cast<double2*>(oth)[t / 2] = make_double2(acc[2 * q], acc[2 * q + 1]);
                { bad.chk(acc[2 * q]); bad.chk(acc[2 * q + 1]); }
            }
        }
    }
    // edges: t in [0, 4) and t > last interior pair end
    const int e0 = tmax >= 4 ? 4 + 2 * ((tmax - 4) / 2) + 2 : 0;  // first t after the interior pairs
    const int lo_n = tmax >= 4 ? 4 : 0;
    const int n_edge = lo_n + (L - e0);
    for (int i = w.lane; i < n_edge; i += 32) {
        const int t = i < lo_n ? i : e0 + (i - lo_n);
        double a = 0.0;
#pragma unroll
        for (int k = 0; k < 7; ++k) {
            int u = t + k - 3;
            u = u < 0 ? 0 : (u > L - 1 ? L - 1 : u);
            a = a + c[k] * cur[u];
        }
        oth[t] = a;
        bad.chk(a);
    }
}

__device__ __forceinline__ bool op_convolve(const DevStage& st, const double* aux, double*& cur, double*& oth, int L, Warp& w, Finite& bad) {
    const double* taps = aux + st.aux_off;
    const int S = st.aux_len, h = S / 2;
    if (S == 7 && ((reinterpret_cast<uintptr_t>(cur) | reinterpret_cast<uintptr_t>(oth)) & 15u) == 0) {
        convolve7(taps, cur, oth, L, w, bad);
        __syncwarp();
        swapbuf(cur, oth);
        return false;
    }
    const int t_hi = L - S + h;  // outputs t in [h, t_hi] read only cur[0 .. L-1]
    for (int t0 = 0; t0 < L; t0 += 128) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        if (t0 >= h && t0 + 127 <= t_hi) {  // warp-uniform interior chunk
            const double* pa = cur + t0 + w.lane - h;
            for (int k = 0; k < S; ++k) {
                const double c = taps[k];
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[q] = acc[q] + c * pa[k + 32 * q];
            }
        } else {
            for (int k = 0; k < S; ++k) {
                const double c = taps[k];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    int u = t0 + w.lane + 32 * q + k - h;
                    u = u < 0 ? 0 : (u > L - 1 ? L - 1 : u);
                    acc[q] = acc[q] + c * cur[u];
                }
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int t = t0 + w.lane + 32 * q;
            if (t < L) {
                oth[t] = acc[q];
                bad.chk(acc[q]);
            }
        }
    }
    __syncwarp();
    swapbuf(cur, oth);
    return false;
}

// BASELINE M5 SpeedWarp.  Two passes over the row: (1) warped positions
// tau_t segment by segment (loop-free per element; written to `oth` as
// scratch), (2) the interpolation of x at tau_t, written back in place
// over tau_t by the same lane.
__device__ __forceinline__ int seg_start(int m, int L, int K) {  // (m L + K) // (K + 1)
    const int64_t num = (int64_t)m * L + K;
    return num <= 0x7fffffff ? (int)((uint32_t)num / (uint32_t)(K + 1)) : (int)(num / (K + 1));
}
__device__ __forceinline__ bool op_speed_warp(const DevStage& st, WStream& s, double*& cur, double*& oth, int L, Warp& w, Finite& bad) {
    const int K = (int)st.i[0];
    const double R = st.f[0];
    if (K == 0 || R == 1.0) return false;
    const int segs = K + 1;
    double* speeds = w.small;
    double* base = w.small + segs;
    int* sbt = reinterpret_cast<int*>(w.iscr);  // segment starts sb[m], m <= K; sb[K + 1] = L
    const double lo = 1.0, range = R - lo;
    for (int m = 0; m < segs; ++m) {
        double v = lo + range * next_double(s, w.lane);
        if (w.lane == 0) speeds[m] = v;
    }
    for (int m = w.lane; m <= K + 1; m += 32) sbt[m] = m <= K ? seg_start(m, L, K) : L;
    __syncwarp();
    if (w.lane == 0) {
        double acc = 0.0;
        base[0] = 0.0;
        for (int m = 0; m < K; ++m) {
            acc = acc + speeds[m] * (double)(sbt[m + 1] - sbt[m]);
            base[m + 1] = acc;
        }
    }
    __syncwarp();
    const double f = ((double)L - 1.0) / ([&] {
        int mm = 0;
        while (mm < K && L - 1 >= sbt[mm + 1]) ++mm;
        return base[mm] + speeds[mm] * (double)(L - 1 - sbt[mm]);
    }());
    // (1) tau_t = (base[m] + speed[m] (t - sb[m])) f on segment m; tau_{L-1} = L - 1
    for (int m = 0; m <= K; ++m) {
        const int sbm = sbt[m], sn = sbt[m + 1];
        const double bm = base[m], spm = speeds[m];
#pragma unroll 4
        for (int t = sbm + w.lane; t < sn; t += 32) oth[t] = (t == L - 1) ? (double)L - 1.0 : (bm + spm * (double)(t - sbm)) * f;
    }
    __syncwarp();
    // (2) Catmull-Rom (or linear) interpolation at tau_t, four per lane step
    const bool cubic = st.i[1] != 0;
    const double x0 = cur[0], xl = cur[L - 1];
    for (int t0 = w.lane; t0 < L; t0 += 128) {
        double taus[4], ys[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int t = t0 + 32 * q;
            taus[q] = oth[t < L ? t : L - 1];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double tau = taus[q];
            int j = (int)floor(tau);
            j = max(0, min(j, L - 2));
            const double fr = tau - (double)j;
            const double p1 = cur[j], p2 = cur[j + 1];
            double y;
            if (cubic) {
                const double p0 = cur[max(j - 1, 0)], p3 = cur[min(j + 2, L - 1)];
                const double a = ((-0.5 * p0 + 1.5 * p1) - 1.5 * p2) + 0.5 * p3;
                const double b = ((p0 - 2.5 * p1) + 2.0 * p2) - 0.5 * p3;
                const double c = -0.5 * p0 + 0.5 * p2;
                y = ((a * fr + b) * fr + c) * fr + p1;
            } else {
                y = p1 + (p2 - p1) * fr;
            }
            y = (tau >= (double)(L - 1)) ? xl : y;
            y = (tau <= 0.0) ? x0 : y;
            ys[q] = y;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int t = t0 + 32 * q;
            if (t < L) {
                oth[t] = ys[q];
                bad.chk(ys[q]);
            }
        }
    }
    __syncwarp();
    swapbuf(cur, oth);
    return false;
}

__device__ __forceinline__ bool spectral_noop(const DevStage& st) {
    if (st.op == SA_OP_APP) return st.f[0] == 0.0 && st.f[1] == 0.0;
    if (st.op == SA_OP_FREQ_MASK) return st.i[0] == 0;
    return st.f[0] == 0.0;  // SINUSOID
}

// sin and cos of a phase perturbation: Taylor series to x^17 / x^18 (Horner
// in x^2, explicit FMA; truncation < 1e-19 for |x| <= pi/4).  APP phases are
// sigma_phase * N(0, 1); larger ones take CUDA's sincos (app_bin_slow).
__device__ __forceinline__ void sincos_small(double x, double* sn, double* cs) {  // |x| <= pi/4
    const double x2 = x * x;
    double ps = 1.0 / 355687428096000.0;
    ps = fma(ps, x2, -1.0 / 1307674368000.0);
    ps = fma(ps, x2, 1.0 / 6227020800.0);
    ps = fma(ps, x2, -1.0 / 39916800.0);
    ps = fma(ps, x2, 1.0 / 362880.0);
    ps = fma(ps, x2, -1.0 / 5040.0);
    ps = fma(ps, x2, 1.0 / 120.0);
    ps = fma(ps, x2, -1.0 / 6.0);
    *sn = fma(x * x2, ps, x);
    double pc = -1.0 / 6402373705728000.0;
    pc = fma(pc, x2, 1.0 / 20922789888000.0);
    pc = fma(pc, x2, -1.0 / 87178291200.0);
    pc = fma(pc, x2, 1.0 / 479001600.0);
    pc = fma(pc, x2, -1.0 / 3628800.0);
    pc = fma(pc, x2, 1.0 / 40320.0);
    pc = fma(pc, x2, -1.0 / 720.0);
    pc = fma(pc, x2, 1.0 / 24.0);
    pc = fma(pc, x2, -0.5);
    *cs = fma(x2, pc, 1.0);
}

// One interior APP bin (freqaugment.py:117-122): r' = max(|X| + amp, 0) at
// angle atan2(im, re) + ph, evaluated as a rotation of X by ph scaled by
// r'/|X| (the same quantity up to rounding; spectral results are compared to
// tolerance).  Common case: |X| and 1/|X| from one rsqrt (|X|^2 comfortably
// normal) and the series sincos (|ph| <= pi/4); otherwise the reference's form.
__device__ __noinline__ double2 app_bin_slow(double2 v, double a, double p) {
    const double r = hypot(v.x, v.y);
    double rn = r + a;
    rn = (rn >= 0.0) ? rn : ((rn != rn) ? rn : 0.0);
    double sn, cs;
    if (r > 0.0) {
        sincos(p, &sn, &cs);
        const double f = rn / r;
        return make_double2(f * (v.x * cs - v.y * sn), f * (v.x * sn + v.y * cs));
    }
    sincos(atan2(v.y, v.x) + p, &sn, &cs);
    return make_double2(rn * cs, rn * sn);
}
__device__ __forceinline__ double2 app_bin(double2 v, double a, double p) {
    const double q = fma(v.x, v.x, v.y * v.y);
    const bool fast = q > 1e-290 && q < 1e290 && fabs(p) <= 0.78539816339744828;
    const double inv_r = rsqrt(q);
    const double r = q * inv_r;
    double rn = r + a;
    rn = (rn >= 0.0) ? rn : ((rn != rn) ? rn : 0.0);
    double sn, cs;
    sincos_small(p, &sn, &cs);
    const double f = rn * inv_r;
    const double2 y = make_double2(f * (v.x * cs - v.y * sn), f * (v.x * sn + v.y * cs));
    return fast ? y : app_bin_slow(v, a, p);
}

// freqaugment.py:106-170 (+ BASELINE M6): perturb the half spectrum X[0..bins)
// (interleaved complex, smem); scratch holds >= 2 * bins doubles.
__device__ __forceinline__ void perturb_spectrum(const DevStage& st, WStream& s, double2* X, int L, double* scratch, Warp& w) {
    const int bins = L / 2 + 1;
    if (st.op == SA_OP_APP) {
        const double sa = st.f[0], sp = st.f[1];
        double* amp = scratch;
        const bool even = (L % 2 == 0);
        const int hi = even ? bins - 1 : bins;
        double* ph = scratch + bins;  // scratch holds >= 2 * bins doubles
        // `bins` magnitude normals then `bins` phase normals (freqaugment.py:
        // 113-114): consecutive draws of one stream, taken in one walk;
        // ph = amp + bins, so draw k lands at scratch[k]; numpy's scaling
        // loc + scale * z (0.0 + sigma * z) is applied where the draws are used
        normals(s, w.lane, 2 * bins, w.zig, [&](int k, double z) { amp[k] = z; });
        __syncwarp();
        // r' = max(|X| + amp, 0) at angle atan2(im, re) + ph (freqaugment.py:
        // 117-122), evaluated as a rotation of X by ph scaled by r'/|X|: the
        // same quantity without atan2 and full-range sin/cos (differs from
        // the reference's formula in rounding only; spectral results are
        // compared to tolerance).  |X| == 0 keeps the reference's form.
        for (int b = 1 + w.lane; b < hi; b += 32) X[b] = app_bin(X[b], 0.0 + sa * amp[b], 0.0 + sp * ph[b]);
        __syncwarp();
        if (w.lane == 0) {
            for (int q = 0; q < (even ? 2 : 1); ++q) {
                int b = q == 0 ? 0 : bins - 1;
                double re = X[b].x;
                double sign = re >= 0 ? 1.0 : -1.0;
                double v = fabs(re) + (0.0 + sa * amp[b]);
                double mv = (v >= 0.0) ? v : 0.0;
                X[b] = make_double2(sign * mv, 0.0);
            }
        }
        __syncwarp();
    } else if (st.op == SA_OP_FREQ_MASK) {
        const int wd = (int)st.i[0];
        int c = (int)bounded(s, w.lane, (uint32_t)(bins - 1));
        int start = c - wd / 2;
        if (start < 0) start = 0;
        if (start > bins - wd) start = bins - wd;
        for (int k = start + w.lane; k < start + wd; k += 32) X[k] = make_double2(0.0, 0.0);
        __syncwarp();
    } else {  // SA_OP_SINUSOID
        const int mb = (int)st.i[0];
        const int b = mb + (int)bounded(s, w.lane, (uint32_t)(bins - mb - 1));
        const double phi = (2.0 * 3.14159265358979323846) * next_double(s, w.lane);
        const double A = st.f[0];
        if (w.lane == 0) {
            double2 v = X[b];
            if (b == 0 || (L % 2 == 0 && b == bins - 1)) {
                v.x = v.x + (A * (double)L) * cos(phi);
            } else {
                double h = (A * (double)L) * 0.5;
                v.x = v.x + h * cos(phi);
                v.y = v.y + h * sin(phi);
            }
            X[b] = v;
        }
        __syncwarp();
    }
}

// freqaugment.py:37-47 SpectralAugmenter._apply (time-domain entry)
#ifndef SA_CHAIN_BLUE
#define SA_CHAIN_BLUE true
#endif
__device__ __forceinline__ bool is_spectral_op(int op) {
    return op == SA_OP_APP || op == SA_OP_FREQ_MASK || op == SA_OP_SINUSOID;
}

// rfft -> perturb -> irfft (freqaugment.py:37-47).  `held` != nullptr: the
// row is already held as its half spectrum (the previous stage kept it).
// keep: leave the result as a spectrum in `held` for the next spectral stage
// (no finiteness check of a time-domain row then; the bins are checked).
template <bool ODD>
__device__ __forceinline__ bool op_spectral(const DevStage& st, WStream& s, double*& cur, double*& oth, int L, Warp& w,
                                            double2*& held, bool keep, Finite& bad) {
    if (spectral_noop(st)) return false;
    // A lone FrequencyMask / RandomSinusoid on an even-length row touches a
    // few bins: its parameters are drawn first (the same draws, in the same
    // order, as perturb_spectrum), and the split, the stage and the fold run
    // only on the bin pairs (k, M - k) it reaches.  Elsewhere fold(split(Z))
    // = conj(Z) (irfft(rfft(x)) = x), the inverse FFT's input directly.  Same
    // formulas and pins as rfft_any / _apply / irfft_any; one call site per
    // transform direction either way (the FFT code is emitted once).
    if (st.op == SA_OP_SINUSOID && !held && !keep) {
        // A lone RandomSinusoid: irfft(X + add e_b) = irfft(X) + irfft(add e_b)
        // and irfft(rfft(x)) = x, so the stage adds bin b's sinusoid in the
        // time domain -- A cos(2 pi b t / L + phi) (interior b: 2 Re(add
        // e^{2 pi i b t / L}) / L with add = (A L / 2) e^{i phi}; DC and
        // Nyquist: the real part only) -- with the same draws, cos / sin of
        // 2 pi b t / L from the W_L table (exact index (b t) mod L), no
        // transform.  Differs from the reference's round trip by its FFT
        // rounding only (spectral tolerance).
        const int bins = L / 2 + 1;
        const int mb = (int)st.i[0];
        const int b = mb + (int)bounded(s, w.lane, (uint32_t)(bins - mb - 1));
        const double phi = (2.0 * 3.14159265358979323846) * next_double(s, w.lane);
        const double A = st.f[0];
        const double cph = cos(phi), sph = sin(phi);
        if (b == 0 || ((L & 1) == 0 && b == bins - 1)) {
            const double c0 = A * cph;
            for (int t = w.lane; t < L; t += 32) {
                const double v = cur[t] + ((b != 0 && (t & 1)) ? -c0 : c0);
                cur[t] = v;
                bad.chk(v);
            }
        } else {
            const int step = (int)((32ll * b) % L);
            int m = (int)(((int64_t)b * w.lane) % L);
            for (int t = w.lane; t < L; t += 32) {
                const double2 e = __ldg(&st.tw[m]);  // (cos, -sin) of 2 pi m / L
                const double v = cur[t] + A * (cph * e.x + sph * e.y);
                cur[t] = v;
                bad.chk(v);
                m += step;
                m = m >= L ? m - L : m;
            }
        }
        __syncwarp();
        return false;
    }
    const bool sparse = !held && !keep && (L & 1) == 0 && st.op != SA_OP_APP;
    const int M = L >> 1;
    int pos = 0, end = 0;
    double2 add = make_double2(0.0, 0.0);
    if (sparse) {
        const int bins = M + 1;
        if (st.op == SA_OP_FREQ_MASK) {
            const int wd = (int)st.i[0];
            int c = (int)bounded(s, w.lane, (uint32_t)(bins - 1));
            pos = c - wd / 2;
            if (pos < 0) pos = 0;
            if (pos > bins - wd) pos = bins - wd;
            end = pos + wd;
        } else {  // SA_OP_SINUSOID
            const int mb = (int)st.i[0];
            pos = mb + (int)bounded(s, w.lane, (uint32_t)(bins - mb - 1));
            end = pos + 1;
            const double phi = (2.0 * 3.14159265358979323846) * next_double(s, w.lane);
            const double A = st.f[0];
            if (pos == 0 || pos == M) {
                add.x = (A * (double)L) * cos(phi);
            } else {
                const double h = (A * (double)L) * 0.5;
                add = make_double2(h * cos(phi), h * sin(phi));
            }
        }
    }
    double2* X;
    if (held) {
        X = held;
        held = nullptr;
        if (w.lane == 0) {  // the pins _apply puts on every fresh rfft
            X[0].y = 0.0;
            if ((L & 1) == 0) X[L / 2].y = 0.0;
        }
        __syncwarp();
    } else {
        X = rfft_any<SA_CHAIN_BLUE && ODD, false, ODD>(cur, oth, L, st.fft, st.tw, w.lane, !sparse);  // sparse: X = the packed Z
    }
    double* free_buf = (reinterpret_cast<double*>(X) == cur) ? oth : cur;
    if (sparse) {
        double2* Y = reinterpret_cast<double2*>(free_buf);
        const bool mask = st.op == SA_OP_FREQ_MASK;
        for (int k = w.lane; k < M; k += 32) {
            const int kc = M - k;  // k = 0 pairs with the Nyquist bin M
            const bool ak = k >= pos && k < end, ac = kc >= pos && kc < end;
            if (!ak && !ac) {
                const double2 z = X[k];
                Y[k] = make_double2(z.x, -z.y);
                continue;
            }
            const double2 zk = X[k], zc = X[k == 0 ? 0 : kc];
            double2 a = cta_split(zk, zc, __ldg(&st.tw[k]));
            double2 c = cta_split(zc, zk, __ldg(&st.tw[kc]));
            if (k == 0) {  // DC / Nyquist imaginary parts pinned (freqaugment.py:40-45)
                a.y = 0.0;
                c.y = 0.0;
            }
            if (mask) {
                if (ak) a = make_double2(0.0, 0.0);
                if (ac) c = make_double2(0.0, 0.0);
            } else {
                if (ak) a = make_double2(a.x + add.x, a.y + add.y);
                if (ac) c = make_double2(c.x + add.x, c.y + add.y);
            }
            Y[k] = cta_fold(a, c, __ldg(&st.tw[k]), k == 0);
        }
        __syncwarp();
    } else {
        perturb_spectrum(st, s, X, L, free_buf, w);
        if (keep) {
            held = X;
            for (int k = w.lane; k < L / 2 + 1; k += 32) { bad.chk(X[k].x); bad.chk(X[k].y); }
            return false;
        }
    }
    // sparse: the folded input is in free_buf and X is scratch
    double2* other = reinterpret_cast<double2*>(free_buf);
    bool ybad = false;
    double* y = irfft_any<SA_CHAIN_BLUE && ODD, false, ODD>(X, other, L, st.fft, st.tw, w.lane, &ybad, sparse);  // checks its outputs
    bad.merge(ybad);
    if (y != cur) swapbuf(cur, oth);
    return false;
}

}  // namespace sa
