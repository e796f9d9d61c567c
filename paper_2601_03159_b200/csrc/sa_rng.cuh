// sa_rng.cuh -- numpy-exact random streams on the device, one warp per stream.
//
// Reference: every draw of the reference comes from
// np.random.Generator(np.random.Philox(key)) with key = derive_stream(
// master_seed, stage j, series i) (reference core.py:71-82).  This file
// restates, for sm_100a, numpy 2.3.5's Philox4x64-10 bit generator and the
// Generator primitives the reference calls (random / normal / uniform /
// integers / permutation / choice), bit-for-bit:
//
//   * Philox is counter based: block b of a fresh stream is philox(key,
//     counter = b + 1) and yields words 4b..4b+3.  A warp therefore fills a
//     128-word WINDOW with one block per lane, in parallel.
//   * 32-bit draws (integers / permutation / choice) use numpy's buffered
//     upper half: a 64-bit word serves two 32-bit draws, low half first, and
//     the buffered half survives intervening 64-bit draws.
//   * The ziggurat normal consumes a data-dependent number of words (one on
//     the fast path, 99.3%; more on the wedge / tail paths).  normals()
//     parses a whole window in one pass: which words head a draw follows
//     from the parity of the slow-word run before them, wedge tests run in
//     parallel, and a warp scan of the accepted heads gives each normal its
//     output index; tails (log1p loop) are resolved uniformly by all lanes
//     with the reference's exact arithmetic.
//
// Every lane of the warp holds an identical copy of the stream state (all
// control flow on it is warp-uniform); only emitted values are lane-private.
// FP expressions are written in the reference's evaluation order and the
// translation unit is compiled with -fmad=false (no FMA contraction).
// The ziggurat TAIL (idx 0 and rabs >= ki[0], 2.6e-4 of normals) evaluates
// log1p: sa_log1p (sa_log1p.h) restates the reference libm's log1p bit for
// bit, so tail normals are bitwise too.  The wedge test compares against exp();
// CUDA's exp and glibc's may differ by an ulp, which changes the decision only
// when the left side equals one of the two candidates exactly (~2^-52 per
// wedge test).
#pragma once
#include <stdint.h>
#include "sa_log1p.h"
#include "zig_tables.h"

#define SA_FULL 0xffffffffu
#define SA_WIN 128  // words per window (32 lanes x 4 words per Philox block)

namespace sa {

struct ZigEntry {  // packed fast-path table: one 16 B load per word
    uint64_t ki;
    double wi;
};

// Device copies of numpy's tables (filled once by sa_init, csrc/sa_capi.cu).
__device__ ZigEntry g_zig[256];
__device__ double g_fi[256];

static constexpr double kZigR = 3.6541528853610088;
static constexpr double kZigInvR = 0.27366123732975828;
static constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // core.py:40-45
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// core.py:77-82
__device__ __forceinline__ void derive_key(uint64_t seed, uint64_t j, uint64_t i, uint64_t& k0,
                                           uint64_t& k1) {
    uint64_t s = mix64(seed);
    s = mix64(s + kGolden + j);
    s = mix64(s + kGolden + i);
    k0 = mix64(s);
    k1 = mix64(s + kGolden);
}

// 64x64 -> 128 multiply from four 32x32->64 IMAD.WIDE products.
__device__ __forceinline__ void mulhilo64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
    lo = a * b;
    hi = __umul64hi(a, b);
}

// numpy Philox4x64-10: Random123 round, Weyl key schedule.
__device__ __forceinline__ void philox(uint64_t k0, uint64_t k1, uint64_t ctr0, uint64_t& o0,
                                       uint64_t& o1, uint64_t& o2, uint64_t& o3) {
    uint64_t c0 = ctr0, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B97F4A7C15ULL;
            k1 += 0xBB67AE8584CAA73BULL;
        }
        uint64_t hi0, lo0, hi1, lo1;
        mulhilo64(0xD2E7470EE14C6C93ULL, c0, hi0, lo0);
        mulhilo64(0xCA5A826395121157ULL, c2, hi1, lo1);
        uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    o0 = c0; o1 = c1; o2 = c2; o3 = c3;
}

// Words 4b..4b+3 of a stream = Philox block counter b + 1.  Test builds
// (tests/csrc/rng_probe.cu) substitute a word array here to drive the window
// walks through crafted streams (wedge / tail runs the generator makes rare).
#ifndef SA_WINDOW_BLOCK
#define SA_WINDOW_BLOCK(k0, k1, b, o0, o1, o2, o3) philox(k0, k1, (b) + 1, o0, o1, o2, o3)
#endif

__device__ __forceinline__ double u53(uint64_t w) {  // Generator.random()
    return (double)(w >> 11) * (1.0 / 9007199254740992.0);
}

// (double)v for v < 2^52 without I2F.F64.U64: splice v into the mantissa of
// 2^52 and subtract 2^52 (exact: both are integers below 2^53).
__device__ __forceinline__ double u52_to_double(uint64_t v) {
    return __longlong_as_double((long long)(v | 0x4330000000000000ULL)) - 4503599627370496.0;
}
// x with its sign bit XORed by bit 8 of the ziggurat word (numpy's
// `sign ? -x : x`; x >= 0 here, so the XOR is the negation, -0.0 included).
__device__ __forceinline__ double zig_signed(double x, uint64_t w) {
    return __longlong_as_double(__double_as_longlong(x) ^ (long long)((w << 55) & 0x8000000000000000ULL));
}
// Two consecutive window words (16-byte aligned) by a shared-memory load: the
// window and the cached gate block both live in shared memory.
__device__ __forceinline__ ulonglong2 lds_u64x2(const uint64_t* p) {
    ulonglong2 v;
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];"
                 : "=l"(v.x), "=l"(v.y)
                 : "r"((uint32_t)__cvta_generic_to_shared(p))
                 : "memory");
    return v;
}

// Warp-uniform stream state.  `win` points at the words currently buffered:
// either the 4 words of block 0 cached by the gate pre-pass (wn = 4) or the
// warp's 128-word window (wn = SA_WIN).
struct WStream {
    uint64_t k0, k1;
    uint64_t wpos;  // absolute index of the next 64-bit word
    uint64_t wb;    // absolute index of win[0]
    uint32_t wn;
    uint32_t has32, u32;
    const uint64_t* win;
    uint64_t* winbuf;  // the warp's window storage (SA_WIN words, smem)
};

// Fill `winbuf` with the 32 Philox blocks blk0 .. blk0+31 (one per lane).
// Out of line (one copy of the unrolled rounds); takes plain values so the
// caller's stream state stays in registers.
__device__ __noinline__ void fill_window(uint64_t k0, uint64_t k1, uint64_t blk0, uint64_t* winbuf, int lane) {
    uint64_t o0, o1, o2, o3;
    SA_WINDOW_BLOCK(k0, k1, blk0 + (uint64_t)lane, o0, o1, o2, o3);
    __syncwarp();  // every lane is done reading the previous window
    ulonglong2* w2 = reinterpret_cast<ulonglong2*>(winbuf) + 2 * lane;
    w2[0] = make_ulonglong2(o0, o1);
    w2[1] = make_ulonglong2(o2, o3);
    __syncwarp();
}

// Refill the window with the 32 blocks starting at the block holding wpos.
__device__ __forceinline__ void refill(WStream& s, int lane) {
    uint64_t blk0 = s.wpos >> 2;
    fill_window(s.k0, s.k1, blk0, s.winbuf, lane);
    s.win = s.winbuf;
    s.wb = blk0 << 2;
    s.wn = SA_WIN;
}

__device__ __forceinline__ uint64_t next64(WStream& s, int lane) {
    if (s.wpos >= s.wb + s.wn) refill(s, lane);
    uint64_t v = s.win[s.wpos - s.wb];
    s.wpos += 1;
    return v;
}

__device__ __forceinline__ uint32_t next32(WStream& s, int lane) {
    if (s.has32) {
        s.has32 = 0;
        return s.u32;
    }
    uint64_t v = next64(s, lane);
    s.has32 = 1;
    s.u32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
}

__device__ __forceinline__ double next_double(WStream& s, int lane) { return u53(next64(s, lane)); }

// One thread's private stream (the CTA spectral kernel draws each stage's
// few scalars on one lane): the same numpy semantics as WStream's scalar
// draws -- block b = philox(key, b + 1), buffered upper 32-bit halves.
struct SStream {
    uint64_t k0, k1, wpos, blk;
    uint64_t w0, w1, w2, w3;
    uint32_t has32, u32;
};
__device__ __forceinline__ void s_init(SStream& s, uint64_t k0, uint64_t k1) {
    s.k0 = k0; s.k1 = k1; s.wpos = 0; s.blk = ~0ull; s.has32 = 0; s.u32 = 0;
}
__device__ __forceinline__ uint64_t s_next64(SStream& s) {
    const uint64_t b = s.wpos >> 2;
    if (b != s.blk) {
        philox(s.k0, s.k1, b + 1, s.w0, s.w1, s.w2, s.w3);
        s.blk = b;
    }
    const uint32_t q = (uint32_t)(s.wpos & 3);
    s.wpos += 1;
    return q == 0 ? s.w0 : (q == 1 ? s.w1 : (q == 2 ? s.w2 : s.w3));
}
__device__ __forceinline__ uint32_t s_next32(SStream& s) {
    if (s.has32) {
        s.has32 = 0;
        return s.u32;
    }
    const uint64_t v = s_next64(s);
    s.has32 = 1;
    s.u32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
}
__device__ __forceinline__ double s_next_double(SStream& s) { return u53(s_next64(s)); }
__device__ __forceinline__ uint32_t s_bounded(SStream& s, uint32_t rng) {  // = bounded()
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFu) return s_next32(s);
    const uint32_t ex = rng + 1u;
    uint64_t m = (uint64_t)s_next32(s) * ex;
    uint32_t left = (uint32_t)m;
    if (left < ex) {
        const uint32_t th = (0u - ex) % ex;
        while (left < th) {
            m = (uint64_t)s_next32(s) * ex;
            left = (uint32_t)m;
        }
    }
    return (uint32_t)(m >> 32);
}

// Generator.integers(0, rng + 1): numpy random_bounded_uint64, 32-bit Lemire.
__device__ __forceinline__ uint32_t bounded(WStream& s, int lane, uint32_t rng) {
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFu) return next32(s, lane);
    uint32_t ex = rng + 1u;
    uint64_t m = (uint64_t)next32(s, lane) * ex;
    uint32_t left = (uint32_t)m;
    if (left < ex) {
        uint32_t th = (0u - ex) % ex;
        while (left < th) {
            m = (uint64_t)next32(s, lane) * ex;
            left = (uint32_t)m;
        }
    }
    return (uint32_t)(m >> 32);
}

// numpy random_interval (masked rejection), used by Generator.permutation.
__device__ __forceinline__ uint32_t interval(WStream& s, int lane, uint32_t max) {
    if (max == 0) return 0;
    uint32_t mask = max;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4; mask |= mask >> 8; mask |= mask >> 16;
    uint32_t v;
    while ((v = (next32(s, lane) & mask)) > max) {
    }
    return v;
}

// Slow path of the ziggurat for a word that failed the fast test (wedge or
// tail, reference numpy random_standard_normal): returns true and the value
// if a normal is produced (else the caller retries with the next word).
// Out of line and rare; the stream travels by value so callers keep theirs
// in registers.
struct ZigSlow {
    WStream s;
    double v;
    bool ok;
};
__device__ __noinline__ void zig_slow_impl(WStream s, int lane, uint64_t r0, ZigSlow* res) {
    int idx = (int)(r0 & 0xff);
    uint64_t r = r0 >> 8;
    int sign = (int)(r & 1);
    uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = (double)rabs * g_zig[idx].wi;
    if (sign) x = -x;
    res->ok = false;
    if (idx == 0) {
        for (;;) {
            double xx = -kZigInvR * sa_log1p(-next_double(s, lane));
            double yy = -sa_log1p(-next_double(s, lane));
            if (yy + yy > xx * xx) {
                res->v = ((rabs >> 8) & 1) ? -(kZigR + xx) : kZigR + xx;
                res->ok = true;
                break;
            }
        }
    } else {
        double u = next_double(s, lane);
        if (((g_fi[idx - 1] - g_fi[idx]) * u + g_fi[idx]) < exp(-0.5 * x * x)) {
            res->v = x;
            res->ok = true;
        }
    }
    res->s = s;
}
__device__ __forceinline__ bool zig_slow(WStream& s, int lane, uint64_t r0, double& out) {
    ZigSlow res;
    zig_slow_impl(s, lane, r0, &res);
    s = res.s;
    out = res.v;
    return res.ok;
}

// One standard normal, warp-uniform (all lanes get the same value).
__device__ __forceinline__ double std_normal(WStream& s, int lane) {
    for (;;) {
        uint64_t r0 = next64(s, lane);
        int idx = (int)(r0 & 0xff);
        uint64_t r = r0 >> 8;
        uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
        ZigEntry ze = g_zig[idx];
        if (rabs < ze.ki) {
            double x = (double)rabs * ze.wi;
            return (r & 1) ? -x : x;
        }
        double v;
        if (zig_slow(s, lane, r0, v)) return v;
    }
}

// Inline window refill for the bulk walks (the Philox rounds are emitted
// once per walk instantiation; scalar draws use the out-of-line refill).
__device__ __forceinline__ void refill_inline(WStream& s, int lane) {
    const uint64_t blk0 = s.wpos >> 2;
    uint64_t o0, o1, o2, o3;
    SA_WINDOW_BLOCK(s.k0, s.k1, blk0 + (uint64_t)lane, o0, o1, o2, o3);
    __syncwarp();
    ulonglong2* w2 = reinterpret_cast<ulonglong2*>(s.winbuf) + 2 * lane;
    w2[0] = make_ulonglong2(o0, o1);
    w2[1] = make_ulonglong2(o2, o3);
    __syncwarp();
    s.win = s.winbuf;
    s.wb = blk0 << 2;
    s.wn = SA_WIN;
}

// numpy's wedge test for slow word w (idx != 0, x its signed value) with
// uniform word uw: accept iff fi[idx] + (fi[idx-1] - fi[idx]) * u < exp(-x^2/2).
// float pre-test: __expf is within ~1e-6 relative of exp(e2); only near-ties
// fall back to the double exp the reference compares with.
__device__ __forceinline__ bool zig_wedge_accept(uint64_t w, double x, uint64_t uw) {
    const int idx = (int)(w & 0xff);
    const double u = u53(uw);
    const double fi0 = __ldg(&g_fi[idx - 1]), fi1 = __ldg(&g_fi[idx]);
    const double lhs = (fi0 - fi1) * u + fi1;
    const double e2 = -0.5 * x * x;  // |x| < 3.66 on the wedge: e2 > -6.7
    const double ef = (double)__expf((float)e2);
    const double d = lhs - ef;
    return (fabs(d) > 1e-5 * ef) ? (d < 0.0) : (lhs < exp(e2));
}

// `count` standard normals in stream order; emit(k, z) is called exactly
// once per k by exactly one lane (k = normal index 0..count-1).
// zig: the fast-path table (shared memory copy of g_zig).
//
// One pass per window parses numpy's sequential word consumption in
// parallel: a fast word is one normal; a wedge word (slow, idx != 0) takes
// the next word as its uniform and yields a normal or nothing; so a word is
// the HEAD of a draw iff the run of slow words right before it (within the
// parse) has even length.  Every lane classifies its 4 words, gets the run
// entering it from its left neighbour, evaluates its wedge heads, and a warp
// scan of accepted heads gives each normal its output index.  The parse stops
// (sequential resolution, then a new pass) at a tail head (idx 0, log1p
// loop), a wedge head whose uniform lies past the window, or in a lane whose
// 4 words are all slow (the entering run would need more than one neighbour).
// Head bits of a lane's 4 words from its slow bits and the parity of the
// slow run entering it: word r heads a draw iff the run before it is even.
__host__ __device__ constexpr uint64_t zig_head_table(int pin) {
    uint64_t t = 0;
    for (int sl = 0; sl < 16; ++sl) {
        int h = !pin, bits = h;
        for (int r = 1; r < 4; ++r) {
            h = ((sl >> (r - 1)) & 1) ? !h : 1;
            bits |= h << r;
        }
        t |= (uint64_t)bits << (4 * sl);
    }
    return t;
}

template <class Emit>
__device__ __forceinline__ void normals(WStream& s, int lane, int count, const ZigEntry* __restrict__ zig,
                                        Emit&& emit) {
    constexpr uint64_t kHead0 = zig_head_table(0), kHead1 = zig_head_table(1);
    const uint32_t lt = (1u << lane) - 1u;
    int k = 0;
    while (k < count) {
        if (s.wpos >= s.wb + s.wn) refill_inline(s, lane);
        const uint32_t wn = s.wn;
        const uint32_t sp = (uint32_t)(s.wpos - s.wb);
        const uint32_t p0 = 4u * lane;
        uint64_t wv[4];
        if (p0 < wn) {
            const ulonglong2 a = lds_u64x2(s.win + 4 * lane), b = lds_u64x2(s.win + 4 * lane + 2);
            wv[0] = a.x; wv[1] = a.y; wv[2] = b.x; wv[3] = b.y;
        } else {
            wv[0] = wv[1] = wv[2] = wv[3] = 0;
        }
        const uint64_t nx = __shfl_down_sync(SA_FULL, wv[0], 1);  // word p0 + 4
        double z[4];
        uint32_t pres = 0, slow = 0, tail = 0;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint64_t w = wv[r];
            const uint64_t rr = w >> 8;
            const uint64_t rabs = (rr >> 1) & 0x000fffffffffffffULL;
            const ZigEntry ze = zig[w & 0xff];
            z[r] = zig_signed(u52_to_double(rabs) * ze.wi, w);
            const uint32_t pb = (p0 + r - sp < wn - sp) ? 1u : 0u;  // sp <= p < wn
            const uint32_t sb = pb & (rabs < ze.ki ? 0u : 1u);
            pres |= pb << r;
            slow |= sb << r;
            tail |= (sb & ((w & 0xff) == 0 ? 1u : 0u)) << r;
        }
        const uint32_t wedge = slow & ~tail;
        // parity of the slow run entering this lane (trailing run of the left one)
        const uint32_t inv = ~slow & 0xfu;
        const uint32_t trail = inv ? (uint32_t)(__clz(inv) - 28) : 4u;
        uint32_t pin = __shfl_up_sync(SA_FULL, trail, 1) & 1u;
        if (lane == 0) pin = 0;
        const uint32_t head = (uint32_t)(((pin ? kHead1 : kHead0) >> (4 * slow)) & 0xfu) & pres;
        uint32_t stop = head & tail;
        if (slow == 0xfu) stop |= head;
        const uint32_t last = wn - 1u - p0;  // the window's last word, if in this lane
        if (last < 4u) stop |= head & wedge & (1u << last);
        const uint32_t mine = stop ? p0 + (uint32_t)(__ffs(stop) - 1) : 0xffffffffu;
        uint32_t t = __reduce_min_sync(SA_FULL, mine);
        t = t > wn ? wn : t;
        // heads before t: fast heads are normals, wedge heads pass the test
        const uint32_t below = t <= p0 ? 0u : (t - p0 >= 4u ? 0xfu : (1u << (t - p0)) - 1u);
        uint32_t acc = head & below & ~slow;
        uint32_t wh = head & below & wedge;
        while (wh) {
            const int r = __ffs(wh) - 1;
            wh &= wh - 1;
            const uint64_t uw = r == 0 ? wv[1] : (r == 1 ? wv[2] : (r == 2 ? wv[3] : nx));
            const uint64_t w = r == 0 ? wv[0] : (r == 1 ? wv[1] : (r == 2 ? wv[2] : wv[3]));
            const double x = r == 0 ? z[0] : (r == 1 ? z[1] : (r == 2 ? z[2] : z[3]));
            if (zig_wedge_accept(w, x, uw)) acc |= 1u << r;
        }
        // output index of each accepted head: exclusive warp prefix of popc(acc)
        // from three ballots of its bits (c <= 4)
        const uint32_t c = (uint32_t)__popc(acc);
        const uint32_t b0 = __ballot_sync(SA_FULL, c & 1u), b1 = __ballot_sync(SA_FULL, c & 2u),
                       b2 = __ballot_sync(SA_FULL, c & 4u);
        const uint32_t excl = __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt);
        const uint32_t tot = __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
        const uint32_t need = (uint32_t)(count - k);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint32_t e = excl + (uint32_t)__popc(acc & ((1u << r) - 1u));
            if (((acc >> r) & 1u) && e < need) emit(k + (int)e, z[r]);
        }
        if (tot >= need) {  // the last normal ends inside this pass
            uint32_t endp = 0;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const uint32_t e = excl + (uint32_t)__popc(acc & ((1u << r) - 1u));
                if (((acc >> r) & 1u) && e == need - 1) endp = p0 + r + ((slow >> r) & 1u) + 1u;
            }
            s.wpos = s.wb + __reduce_max_sync(SA_FULL, endp);
            return;
        }
        k += (int)tot;
        s.wpos = s.wb + t;
        if (t >= wn) continue;
        // stop head at t, resolved uniformly with the reference's arithmetic
        const uint64_t r0 = s.win[t];
        s.wpos += 1;
        bool ok;
        double v;
        if (r0 & 0xff) {  // wedge (its uniform may start the next window)
            const uint64_t rr = r0 >> 8;
            const uint64_t rabs = (rr >> 1) & 0x000fffffffffffffULL;
            double x = (double)rabs * zig[r0 & 0xff].wi;
            if (rr & 1) x = -x;
            if (s.wpos >= s.wb + s.wn) refill(s, lane);
            const uint64_t uw = s.win[s.wpos - s.wb];
            s.wpos += 1;
            ok = zig_wedge_accept(r0, x, uw);
            v = x;
        } else {
            ok = zig_slow(s, lane, r0, v);  // tail: out of line, ~3e-4 of words
        }
        if (ok) {
            if (lane == 0) emit(k, v);
            k += 1;
        }
    }
}

// `count` doubles random() in stream order; emit(k, u) once per k.
template <class Emit>
__device__ __forceinline__ void doubles(WStream& s, int lane, int count, Emit&& emit) {
    int k = 0;
    while (k < count) {
        if (s.wpos >= s.wb + s.wn) refill_inline(s, lane);
        const uint32_t sp = (uint32_t)(s.wpos - s.wb);
        const uint32_t avail = s.wn - sp;
        const uint32_t take = avail < (uint32_t)(count - k) ? avail : (uint32_t)(count - k);
        if (4u * lane < s.wn) {
            const ulonglong2* w2 = reinterpret_cast<const ulonglong2*>(s.win) + 2 * lane;
            ulonglong2 a = w2[0], b = w2[1];
            const uint64_t wv[4] = {a.x, a.y, b.x, b.y};
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const uint32_t off = 4u * lane + r - sp;
                if (off < take) emit(k + (int)off, u53(wv[r]));
            }
        }
        k += (int)take;
        s.wpos += take;
    }
}

}  // namespace sa
