// sa_text.cuh -- float64 <-> text on the device, bit-exact with CPython.
//
// The reference's dataset files (reference datafiles.py) write every value
// as repr(float(v)) -- CPython's shortest round-trip decimal -- and read
// fields with float(str) -- correctly rounded decimal -> binary64.  This file
// restates both, per element, for the device dataset codec:
//
//  * shortest_decimal(): the shortest digit string that rounds back to the
//    double, closest to it, ties to even (Adams, "Ryu", PLDI 2018): the
//    interval of valid decimals [m2 - 1/2, m2 + 1/2] ulp is scaled by 10^-q
//    with 128-bit fixed-point powers of 5 (sa_text_tables.h, generated
//    exactly), then digits are removed while the interval still contains a
//    shorter number.
//  * repr_format(): CPython's float_repr layout around those digits:
//    exponent form iff decpt <= -4 or decpt > 16 (e[+-]XX, >= 2 digits),
//    otherwise fixed form with at least one fractional digit ("1.0").
//  * parse_pyfloat(): float() grammar ([+-] digits with '_' separators,
//    fraction, exponent, inf / infinity / nan) with correct rounding: a
//    64-bit significand times a 128-bit power of 5 decides the rounding
//    unless the product is within its error bound of a halfway point
//    (Lemire 2021); those cases, and >19-digit or subnormal inputs, are
//    decided exactly by big-integer comparison.
#pragma once
#include <stdint.h>

#include "sa_text_tables.h"

namespace sa {

// ------------------------------------------------------------ 128-bit helpers
struct U128 {
    uint64_t lo, hi;
};
__device__ __forceinline__ U128 mul64(uint64_t a, uint64_t b) { return {a * b, __umul64hi(a, b)}; }

__device__ __forceinline__ int pow5bits(int e) { return ((e * 1217359) >> 19) + 1; }
__device__ __forceinline__ int log10_pow2(int e) { return (e * 78913) >> 18; }
__device__ __forceinline__ int log10_pow5(int e) { return (e * 732923) >> 20; }

// (m * mul) >> j for a 128-bit mul and 64 <= j < 192
__device__ __forceinline__ uint64_t mul_shift(uint64_t m, const uint64_t* mul, int j) {
    const U128 b0 = mul64(m, mul[0]);
    const U128 b2 = mul64(m, mul[1]);
    const uint64_t mid = b0.hi + b2.lo;
    const uint64_t hi = b2.hi + (mid < b0.hi ? 1 : 0);
    const int s = j - 64;
    return s == 0 ? mid : (s < 64 ? ((mid >> s) | (hi << (64 - s))) : (hi >> (s - 64)));
}

__device__ __forceinline__ int pow5_factor(uint64_t v) {
    int c = 0;
    while (v % 5 == 0) {
        v /= 5;
        ++c;
    }
    return c;
}
__device__ __forceinline__ bool multiple_of_pow5(uint64_t v, int p) { return pow5_factor(v) >= p; }
__device__ __forceinline__ bool multiple_of_pow2(uint64_t v, int p) {
    return p >= 64 ? v == 0 : (v & ((1ull << p) - 1)) == 0;
}

// ------------------------------------------------------------ shortest digits
struct Decimal {
    uint64_t digits;  // value = digits * 10^exp10
    int exp10;
};

// Shortest round-trip decimal of a finite, non-zero double.
__device__ Decimal shortest_decimal(uint64_t bits) {
    const uint64_t mant = bits & ((1ull << 52) - 1);
    const int bexp = (int)((bits >> 52) & 0x7ff);
    int e2;
    uint64_t m2;
    if (bexp == 0) {
        e2 = 1 - 1023 - 52 - 2;
        m2 = mant;
    } else {
        e2 = bexp - 1023 - 52 - 2;
        m2 = (1ull << 52) | mant;
    }
    const bool accept_bounds = (m2 & 1) == 0;  // round-half-even parsing accepts the ends
    const uint64_t mv = 4 * m2;
    const uint64_t mm_shift = (mant != 0 || bexp <= 1) ? 1 : 0;  // lower gap halves at powers of two
    const uint64_t up = mv + 2, dn = mv - 1 - mm_shift;

    uint64_t vr, vp, vm;
    int e10;
    bool vm_tz = false, vr_tz = false;
    if (e2 >= 0) {
        const int q = log10_pow2(e2) - (e2 > 3 ? 1 : 0);
        e10 = q;
        const int j = -e2 + q + 125 + pow5bits(q) - 1;
        vr = mul_shift(mv, kRyuPow5Inv[q], j);
        vp = mul_shift(up, kRyuPow5Inv[q], j);
        vm = mul_shift(dn, kRyuPow5Inv[q], j);
        if (q <= 21) {  // the scaled interval ends may be exact integers
            if (mv % 5 == 0) vr_tz = multiple_of_pow5(mv, q);
            else if (accept_bounds) vm_tz = multiple_of_pow5(dn, q);
            else vp -= multiple_of_pow5(up, q) ? 1 : 0;
        }
    } else {
        const int q = log10_pow5(-e2) - (-e2 > 1 ? 1 : 0);
        e10 = q + e2;
        const int i = -e2 - q;
        const int j = q - (pow5bits(i) - 125);
        vr = mul_shift(mv, kRyuPow5[i], j);
        vp = mul_shift(up, kRyuPow5[i], j);
        vm = mul_shift(dn, kRyuPow5[i], j);
        if (q <= 1) {
            vr_tz = true;
            if (accept_bounds) vm_tz = mm_shift == 1;
            else --vp;
        } else if (q < 63) {
            vr_tz = multiple_of_pow2(mv, q);
        }
    }

    int removed = 0;
    uint64_t last = 0;
    uint64_t out;
    if (vm_tz || vr_tz) {
        // general case: track whether the removed digits were all zero
        for (;;) {
            const uint64_t p10 = vp / 10, m10 = vm / 10;
            if (p10 <= m10) break;
            const uint64_t r10 = vr / 10;
            vm_tz = vm_tz && (vm - 10 * m10 == 0);
            vr_tz = vr_tz && (last == 0);
            last = vr - 10 * r10;
            vr = r10; vp = p10; vm = m10;
            ++removed;
        }
        if (vm_tz) {
            for (;;) {
                const uint64_t m10 = vm / 10;
                if (vm - 10 * m10 != 0) break;
                const uint64_t r10 = vr / 10;
                vr_tz = vr_tz && (last == 0);
                last = vr - 10 * r10;
                vr = r10; vp /= 10; vm = m10;
                ++removed;
            }
        }
        if (vr_tz && last == 5 && (vr & 1) == 0) last = 4;  // exact ...50...0: round half even
        out = vr + (((vr == vm) && (!accept_bounds || !vm_tz)) || last >= 5 ? 1 : 0);
    } else {
        bool round_up = false;
        for (;;) {
            const uint64_t p10 = vp / 10, m10 = vm / 10;
            if (p10 <= m10) break;
            const uint64_t r10 = vr / 10;
            round_up = (vr - 10 * r10) >= 5;
            vr = r10; vp = p10; vm = m10;
            ++removed;
        }
        out = vr + ((vr == vm || round_up) ? 1 : 0);
    }
    return {out, e10 + removed};
}

// ------------------------------------------------------------ repr(float)
// CPython's float_repr (mode 'r', Py_DTSF_ADD_DOT_0): shortest digits; the
// exponent form 'd[.ddd]e[+-]XX' iff the decimal point position decpt is
// <= -4 or > 16, else fixed notation with at least one fractional digit.
struct Repr {
    uint64_t digits;
    int nd;     // digit count of `digits`
    int decpt;  // value = 0.digits * 10^decpt
    int kind;   // 0 finite non-zero, 1 zero, 2 inf, 3 nan
    bool neg;
};

__device__ __forceinline__ int digit_count(uint64_t v) {
    int n = 1;
    uint64_t p = 10;
    while (n < 20 && v >= p) {
        ++n;
        p *= 10;
    }
    return n;
}

__device__ __forceinline__ Repr repr_decompose(double v) {
    uint64_t bits = (uint64_t)__double_as_longlong(v);
    Repr r;
    r.neg = (bits >> 63) != 0;
    bits &= ~(1ull << 63);
    r.digits = 0;
    r.nd = 0;
    r.decpt = 0;
    if (bits >= 0x7ff0000000000000ull) {
        r.kind = bits > 0x7ff0000000000000ull ? 3 : 2;
        if (r.kind == 3) r.neg = false;  // nan prints unsigned
        return r;
    }
    if (bits == 0) {
        r.kind = 1;
        return r;
    }
    r.kind = 0;
    const Decimal d = shortest_decimal(bits);
    r.digits = d.digits;
    r.nd = digit_count(d.digits);
    r.decpt = d.exp10 + r.nd;
    return r;
}

__device__ __forceinline__ int repr_len(const Repr& r) {
    int n = r.neg ? 1 : 0;
    if (r.kind != 0) return n + 3;  // "0.0" / "inf" / "nan"
    const int nd = r.nd, decpt = r.decpt;
    if (decpt <= -4 || decpt > 16) {
        const int x = decpt - 1 < 0 ? 1 - decpt : decpt - 1;
        return n + nd + (nd > 1 ? 1 : 0) + 2 + (x >= 100 ? 3 : 2);
    }
    if (decpt <= 0) return n + 2 - decpt + nd;
    if (decpt >= nd) return n + decpt + 2;
    return n + nd + 1;
}

// writes repr_len(r) bytes at dst
__device__ __forceinline__ void repr_write(const Repr& r, char* dst) {
    int n = 0;
    if (r.neg) dst[n++] = '-';
    if (r.kind == 1) {
        dst[n] = '0'; dst[n + 1] = '.'; dst[n + 2] = '0';
        return;
    }
    if (r.kind == 2) {
        dst[n] = 'i'; dst[n + 1] = 'n'; dst[n + 2] = 'f';
        return;
    }
    if (r.kind == 3) {
        dst[n] = 'n'; dst[n + 1] = 'a'; dst[n + 2] = 'n';
        return;
    }
    const int nd = r.nd, decpt = r.decpt;
    // digit k (0 = most significant) lands at pos(k); written from the last
    // digit backwards so each division yields one character
    if (decpt <= -4 || decpt > 16) {
        uint64_t t = r.digits;
        for (int k = nd - 1; k >= 1; --k) {
            const uint64_t q = t / 10;
            dst[n + 1 + k] = (char)('0' + (int)(t - 10 * q));
            t = q;
        }
        dst[n] = (char)('0' + (int)t);
        if (nd > 1) dst[n + 1] = '.';
        n += nd + (nd > 1 ? 1 : 0);
        dst[n++] = 'e';
        int x = decpt - 1;
        dst[n++] = x < 0 ? '-' : '+';
        if (x < 0) x = -x;
        if (x >= 100) dst[n++] = (char)('0' + x / 100);
        dst[n++] = (char)('0' + (x / 10) % 10);
        dst[n++] = (char)('0' + x % 10);
        return;
    }
    if (decpt <= 0) {
        dst[n++] = '0';
        dst[n++] = '.';
        for (int k = 0; k < -decpt; ++k) dst[n++] = '0';
        uint64_t t = r.digits;
        for (int k = nd - 1; k >= 0; --k) {
            const uint64_t q = t / 10;
            dst[n + k] = (char)('0' + (int)(t - 10 * q));
            t = q;
        }
        return;
    }
    if (decpt >= nd) {
        uint64_t t = r.digits;
        for (int k = nd - 1; k >= 0; --k) {
            const uint64_t q = t / 10;
            dst[n + k] = (char)('0' + (int)(t - 10 * q));
            t = q;
        }
        n += nd;
        for (int k = 0; k < decpt - nd; ++k) dst[n++] = '0';
        dst[n] = '.';
        dst[n + 1] = '0';
        return;
    }
    uint64_t t = r.digits;  // digits 0..decpt-1, '.', digits decpt..nd-1
    for (int k = nd - 1; k >= 0; --k) {
        const uint64_t q = t / 10;
        dst[n + k + (k >= decpt ? 1 : 0)] = (char)('0' + (int)(t - 10 * q));
        t = q;
    }
    dst[n + decpt] = '.';
}

// Writes CPython's repr of a double into dst (>= 25 bytes); returns the
// number of bytes.
__device__ __forceinline__ int repr_format(double v, char* dst) {
    const Repr r = repr_decompose(v);
    repr_write(r, dst);
    return repr_len(r);
}

// ------------------------------------------------------------ exact big integers
// Little-endian 32-bit limbs; capacity for ~4000 bits (decimal inputs are
// capped at 800 significant digits + a sticky bit, powers up to 2^1100 * 5^342).
#define SA_BIG_LIMBS 136
struct Big {
    uint32_t w[SA_BIG_LIMBS];
    int n;
};
__device__ __forceinline__ void big_set(Big& b, uint64_t v) {
    b.n = 0;
    while (v) {
        b.w[b.n++] = (uint32_t)v;
        v >>= 32;
    }
}
__device__ __forceinline__ void big_mul_small(Big& b, uint32_t m) {
    uint64_t carry = 0;
    for (int i = 0; i < b.n; ++i) {
        const uint64_t t = (uint64_t)b.w[i] * m + carry;
        b.w[i] = (uint32_t)t;
        carry = t >> 32;
    }
    if (carry && b.n < SA_BIG_LIMBS) b.w[b.n++] = (uint32_t)carry;
}
__device__ __forceinline__ void big_add_small(Big& b, uint32_t a) {
    uint64_t carry = a;
    for (int i = 0; i < b.n && carry; ++i) {
        const uint64_t t = (uint64_t)b.w[i] + carry;
        b.w[i] = (uint32_t)t;
        carry = t >> 32;
    }
    if (carry && b.n < SA_BIG_LIMBS) b.w[b.n++] = (uint32_t)carry;
}
__device__ void big_mul_pow5(Big& b, int e) {
    while (e >= 13) {  // 5^13 < 2^32
        big_mul_small(b, 1220703125u);
        e -= 13;
    }
    uint32_t p = 1;
    while (e-- > 0) p *= 5;
    if (p != 1) big_mul_small(b, p);
}
__device__ void big_shl(Big& b, int s) {
    if (b.n == 0 || s == 0) return;
    const int ws = s / 32, bs = s % 32;
    int n = b.n + ws + 1;
    if (n > SA_BIG_LIMBS) n = SA_BIG_LIMBS;
    for (int i = n - 1; i >= 0; --i) {
        const int src = i - ws;
        uint32_t v = src >= 0 && src < b.n ? b.w[src] << bs : 0;
        if (bs && src - 1 >= 0 && src - 1 < b.n) v |= b.w[src - 1] >> (32 - bs);
        b.w[i] = v;
    }
    b.n = n;
    while (b.n && b.w[b.n - 1] == 0) --b.n;
}
__device__ int big_cmp(const Big& a, const Big& b) {
    if (a.n != b.n) return a.n < b.n ? -1 : 1;
    for (int i = a.n - 1; i >= 0; --i)
        if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
    return 0;
}

// ------------------------------------------------------------ float(str)
__device__ __forceinline__ bool is_digit(char c) { return c >= '0' && c <= '9'; }

// D = the first K significant digits found in s[p0, p1) (skipping '.' / '_')
__device__ void big_from_digits(Big& D, const char* s, int p0, int p1, int K) {
    big_set(D, 0);
    int k = 0;
    uint32_t chunk = 0;
    int cn = 0;
    for (int i = p0; i < p1 && k < K; ++i) {
        if (!is_digit(s[i])) continue;
        chunk = chunk * 10 + (uint32_t)(s[i] - '0');
        ++cn;
        ++k;
        if (cn == 9) {
            big_mul_small(D, 1000000000u);
            big_add_small(D, chunk);
            chunk = 0;
            cn = 0;
        }
    }
    if (cn) {
        uint32_t p = 1;
        for (int t = 0; t < cn; ++t) p *= 10;
        big_mul_small(D, p);
        big_add_small(D, chunk);
    }
}

// sign of D * 10^e10 (+ sticky) - A * 2^a
__device__ int cmp_value(const Big& D, int e10, bool sticky, uint64_t A, int a) {
    Big X = D, Y;
    big_set(Y, A);
    if (e10 >= 0) big_mul_pow5(X, e10);
    else big_mul_pow5(Y, -e10);
    const int lo = e10 < a ? e10 : a;
    big_shl(X, e10 - lo);
    big_shl(Y, a - lo);
    int c = big_cmp(X, Y);
    if (c == 0 && sticky) c = 1;
    return c;
}

__device__ __forceinline__ uint64_t pack_double(uint64_t m, int e2) {
    // m * 2^e2 with m < 2^53; e2 = -1074 and m < 2^52 is subnormal
    if (m == 0) return 0;
    if (e2 + 52 > 1023) return 0x7ff0000000000000ull;
    if (m < (1ull << 52)) return m;  // subnormal (e2 == -1074)
    return ((uint64_t)(e2 + 52 + 1023) << 52) | (m & ((1ull << 52) - 1));
}

// Exact decision by big-integer comparison around the candidate m * 2^e2
// (halfway-close products, > 19 significant digits, subnormals).  Kept out of
// line: the fast path stays small and register-light.
__device__ __noinline__ uint64_t parse_exact(const char* s, int p0, int m1, int nd, long long e_last, int E,
                                             uint64_t mant) {
    const int K = nd < 800 ? nd : 800;
    bool sticky = false;
    {
        int k = 0;
        for (int t = p0; t < m1; ++t) {
            if (!is_digit(s[t])) continue;
            if (k >= K && s[t] != '0') sticky = true;
            ++k;
        }
    }
    const int e10 = (int)(e_last + (nd - K));
    Big D;
    big_from_digits(D, s, p0, m1, K);
    uint64_t m;
    int e2;
    if (E >= -1022) {
        m = mant;
        e2 = E - 52;
    } else {  // subnormal candidate
        const int sh = -1022 - E;
        m = sh >= 64 ? 0 : mant >> sh;
        e2 = -1074;
    }
    for (int it = 0; it < 16; ++it) {  // candidate is within a few ulps
        if (m > 0 && cmp_value(D, e10, sticky, m, e2) < 0) {
            if (m > (1ull << 52) || e2 == -1074) --m;
            else { m = (1ull << 53) - 1; --e2; }
            continue;
        }
        if (cmp_value(D, e10, sticky, m + 1, e2) >= 0) {
            ++m;
            if (m == (1ull << 53)) { m = 1ull << 52; ++e2; }
            continue;
        }
        break;
    }
    const int c = cmp_value(D, e10, sticky, 2 * m + 1, e2 - 1);
    if (c > 0 || (c == 0 && (m & 1))) {
        ++m;
        if (m == (1ull << 53)) { m = 1ull << 52; ++e2; }
    }
    return pack_double(m, e2);
}

__device__ __noinline__ bool parse_special(const char* s, int i, int n, bool neg, double* out) {
    const int len = n - i;
    char w[8];
    if (len != 3 && len != 8) return false;
    for (int k = 0; k < len; ++k) {
        const char c = s[i + k];
        w[k] = (c >= 'A' && c <= 'Z') ? (char)(c + 32) : c;
    }
    const bool inf = (len == 3 && w[0] == 'i' && w[1] == 'n' && w[2] == 'f') ||
                     (len == 8 && w[0] == 'i' && w[1] == 'n' && w[2] == 'f' && w[3] == 'i' && w[4] == 'n' &&
                      w[5] == 'i' && w[6] == 't' && w[7] == 'y');
    const bool nan = len == 3 && w[0] == 'n' && w[1] == 'a' && w[2] == 'n';
    if (!inf && !nan) return false;
    const uint64_t bits = inf ? 0x7ff0000000000000ull : 0x7ff8000000000000ull;
    *out = __longlong_as_double((long long)(bits | (neg ? 1ull << 63 : 0)));
    return true;
}

// CPython float(): [+-] (digits['.'digits] | '.'digits) [e[+-]digits] with
// '_' allowed between two digits, or inf / infinity / nan (case-insensitive).
// s[0..n) is already stripped of surrounding whitespace.  One pass collects
// the first 19 significant digits; the 64x128-bit product decides the
// rounding unless it is too close to a halfway point (parse_exact).
__device__ __noinline__ bool parse_pyfloat(const char* s, int n, double* out) {
    int i = 0;
    bool neg = false;
    if (i < n && (s[i] == '+' || s[i] == '-')) {
        neg = s[i] == '-';
        ++i;
    }
    if (i < n && !is_digit(s[i]) && s[i] != '.') return parse_special(s, i, n, neg, out);
    // mantissa, one pass
    const int m0 = i;
    int ndig = 0, nfrac = 0, nd = 0, p0 = -1;
    bool frac = false, trunc = false;
    uint64_t w19 = 0;
    for (; i < n; ++i) {
        const char c = s[i];
        const unsigned d = (unsigned)(c - '0');
        if (d < 10) {
            ++ndig;
            nfrac += frac;
            if (d != 0 || nd > 0) {
                if (nd == 0) p0 = i;
                if (nd < 19) w19 = w19 * 10 + d;
                else trunc |= d != 0;
                ++nd;
            }
        } else if (c == '_') {
            if (i == m0 || i + 1 >= n || !is_digit(s[i - 1]) || !is_digit(s[i + 1])) return false;
        } else if (c == '.' && !frac) {
            frac = true;
        } else {
            break;
        }
    }
    if (ndig == 0) return false;
    const int m1 = i;
    long long ex = 0;
    if (i < n && (s[i] == 'e' || s[i] == 'E')) {
        ++i;
        bool eneg = false;
        if (i < n && (s[i] == '+' || s[i] == '-')) {
            eneg = s[i] == '-';
            ++i;
        }
        int ed = 0;
        for (; i < n; ++i) {
            const unsigned d = (unsigned)(s[i] - '0');
            if (d < 10) {
                if (ex < 1000000000ll) ex = ex * 10 + d;
                ++ed;
            } else if (s[i] == '_' && ed > 0 && i + 1 < n && is_digit(s[i + 1])) {
                continue;
            } else {
                break;
            }
        }
        if (ed == 0) return false;
        if (eneg) ex = -ex;
    }
    if (i != n) return false;

    const uint64_t sgn = neg ? 1ull << 63 : 0;
    if (nd == 0) {  // all digits zero
        *out = __longlong_as_double((long long)sgn);
        return true;
    }
    // value = (all significant digits as an integer) * 10^(ex - nfrac)
    const long long e_last = ex - nfrac;
    const int n19 = nd < 19 ? nd : 19;
    const long long q_ll = e_last + (nd - n19);  // exponent of w19's last digit
    if (q_ll + n19 <= -324) {                  // < 10^-324: rounds to zero
        *out = __longlong_as_double((long long)sgn);
        return true;
    }
    if (q_ll + n19 - 1 >= 309) {               // >= 10^309: rounds to inf
        *out = __longlong_as_double((long long)(sgn | 0x7ff0000000000000ull));
        return true;
    }
    const int q = (int)q_ll;  // in [-342, 308] here

    // ---- fast path: normalised w19 times the 128-bit power of five
    const int lz = __clzll(w19);
    const uint64_t wn = w19 << lz;
    const uint64_t* T = kLemirePow5[q + 342];
    const U128 a = mul64(wn, T[1]);
    const U128 b = mul64(wn, T[0]);
    uint64_t mid = a.lo + b.hi;
    uint64_t hi = a.hi + (mid < a.lo ? 1 : 0);
    int lead = 191;
    if (!(hi >> 63)) {
        hi = (hi << 1) | (mid >> 63);
        mid = (mid << 1) | (b.lo >> 63);
        lead = 190;
    }
    // T = 5^q * 2^(127 - floor(log2 5^q)) (+-1); value ~ P * 2^(q - lz - s)
    const int fl5 = q >= 0 ? pow5bits(q) - 1 : -pow5bits(-q);
    const int E = lead + q - lz - (127 - fl5);  // unbiased exponent of the leading bit
    const uint64_t mant = hi >> 11;             // 53 bits
    const uint64_t rem = hi & 0x7ff;            // the 139-bit remainder is rem:mid:low
    // |product error| < 2^65 low-units: the rounding is decided unless the
    // remainder lies within 2 mid-units of the halfway pattern 0x400:0:0
    const bool near_half = (rem == 0x400 && mid <= 1) || (rem == 0x3ff && mid >= ~1ull);
    uint64_t bits;
    if (!trunc && !near_half && E >= -1022 && E <= 1023) {
        uint64_t m = mant + ((rem > 0x400 || (rem == 0x400 && mid > 1)) ? 1 : 0);
        int e2 = E - 52;
        if (m == (1ull << 53)) {
            m >>= 1;
            ++e2;
        }
        bits = pack_double(m, e2);
    } else {
        bits = parse_exact(s, p0, m1, nd, e_last, E, mant);
    }
    *out = __longlong_as_double((long long)(sgn | bits));
    return true;
}

// ------------------------------------------------------------ float(str) of one field
// UTF-8 code point at s[i] (valid UTF-8 assumed); returns its byte length.
__device__ __forceinline__ int utf8_decode(const char* s, int64_t i, int64_t n, uint32_t* cp) {
    const uint32_t c = (uint8_t)s[i];
    if (c < 0x80) { *cp = c; return 1; }
    int len = c >= 0xf0 ? 4 : (c >= 0xe0 ? 3 : 2);
    if (i + len > n) len = (int)(n - i);
    uint32_t v = c & (len == 2 ? 0x1f : (len == 3 ? 0x0f : 0x07));
    for (int k = 1; k < len; ++k) v = (v << 6) | ((uint8_t)s[i + k] & 0x3f);
    *cp = v;
    return len;
}

__device__ __forceinline__ bool is_unicode_space(uint32_t cp) {
    for (int k = 0; k < kNumUnicodeSpaces; ++k)
        if (kUnicodeSpaces[k] == cp) return true;
    return false;
}

// value 0..9 of a Unicode decimal digit, -1 otherwise
__device__ __forceinline__ int unicode_decimal(uint32_t cp) {
    int lo = 0, hi = kNumDecimalRuns - 1;
    while (lo < hi) {  // last run start <= cp
        const int mid = (lo + hi + 1) >> 1;
        if (kDecimalRuns[mid] <= cp) lo = mid;
        else hi = mid - 1;
    }
    const uint32_t d = cp - kDecimalRuns[lo];
    return (cp >= kDecimalRuns[lo] && d < 10) ? (int)d : -1;
}

__device__ __forceinline__ bool py_isspace(char c) { return c == ' ' || (c >= 9 && c <= 13); }

// float(text[a:b]) exactly as CPython's float(str): non-ASCII text is first
// mapped (Unicode whitespace -> ' ', Nd digits -> ASCII, anything else
// fails) into scratch[a:...] (same size as text, may be null when the text is
// ASCII), then ASCII whitespace is stripped and the rest parsed.
// Fast path for the common spelling [+-]digits[.digits][(e|E)[+-]d{1,4}]
// with at most 19 digits and no '_': one tight loop, then the 64x128-bit
// product.  Returns false when it cannot decide (other grammar, more digits,
// near-halfway products, subnormal / overflow range); the caller then runs
// the full parser, which gives the same answer for every input it accepts.
__device__ __forceinline__ bool parse_simple(const char* s, int n, double* out) {
    int i = (n > 0 && (s[0] == '-' || s[0] == '+')) ? 1 : 0;
    const bool neg = n > 0 && s[0] == '-';
    uint64_t w = 0;
    int ndig = 0, dot = -1;
    for (; i < n; ++i) {
        const unsigned d = (unsigned)(uint8_t)s[i] - (unsigned)'0';
        if (d < 10) {
            w = w * 10 + d;
            ++ndig;
        } else if (s[i] == '.' && dot < 0) {
            dot = ndig;
        } else {
            break;
        }
    }
    if (ndig == 0 || ndig > 19) return false;
    int ex = 0;
    if (i < n) {
        if ((s[i] | 0x20) != 'e') return false;
        ++i;
        const bool eneg = i < n && s[i] == '-';
        if (i < n && (s[i] == '-' || s[i] == '+')) ++i;
        const int e0 = i;
        for (; i < n; ++i) {
            const unsigned d = (unsigned)(uint8_t)s[i] - (unsigned)'0';
            if (d >= 10) return false;
            ex = ex * 10 + (int)d;
        }
        if (i == e0 || i - e0 > 4) return false;
        if (eneg) ex = -ex;
    }
    const uint64_t sgn = neg ? 1ull << 63 : 0;
    if (w == 0) {
        *out = __longlong_as_double((long long)sgn);
        return true;
    }
    const int q = ex - (dot >= 0 ? ndig - dot : 0);
    if (q < -342 || q > 308) return false;
    const int lz = __clzll(w);
    const uint64_t wn = w << lz;
    const uint64_t* T = kLemirePow5[q + 342];
    const U128 a = mul64(wn, T[1]);
    const U128 b = mul64(wn, T[0]);
    uint64_t mid = a.lo + b.hi;
    uint64_t hi = a.hi + (mid < a.lo ? 1 : 0);
    int lead = 191;
    if (!(hi >> 63)) {
        hi = (hi << 1) | (mid >> 63);
        mid = (mid << 1) | (b.lo >> 63);
        lead = 190;
    }
    const int fl5 = q >= 0 ? pow5bits(q) - 1 : -pow5bits(-q);
    const int E = lead + q - lz - (127 - fl5);
    const uint64_t rem = hi & 0x7ff;
    const bool near_half = (rem == 0x400 && mid <= 1) || (rem == 0x3ff && mid >= ~1ull);
    if (near_half || E < -1022 || E > 1023) return false;
    uint64_t m = (hi >> 11) + ((rem > 0x400 || (rem == 0x400 && mid > 1)) ? 1 : 0);
    int e2 = E - 52;
    if (m == (1ull << 53)) {
        m >>= 1;
        ++e2;
    }
    *out = __longlong_as_double((long long)(sgn | pack_double(m, e2)));
    return true;
}

__device__ __noinline__ bool parse_field_unicode(const char* text, int64_t a, int64_t b, char* scratch,
                                                 double* out) {
    int64_t w = a;
    for (int64_t p = a; p < b;) {
        uint32_t cp;
        const int k = utf8_decode(text, p, b, &cp);
        p += k;
        char c;
        if (cp < 127) c = (char)cp;
        else if (is_unicode_space(cp)) c = ' ';
        else {
            const int d = unicode_decimal(cp);
            if (d < 0) return false;
            c = (char)('0' + d);
        }
        scratch[w++] = c;
    }
    b = w;
    while (a < b && py_isspace(scratch[a])) ++a;
    while (b > a && py_isspace(scratch[b - 1])) --b;
    if (b - a > 0x7fffffff) return false;
    return parse_pyfloat(scratch + a, (int)(b - a), out);
}

__device__ bool parse_field(const char* text, int64_t a, int64_t b, char* scratch, double* out) {
    int64_t s = a, e = b;
    while (s < e && py_isspace(text[s])) ++s;
    while (e > s && py_isspace(text[e - 1])) --e;
    if (e - s <= 0x7fffffff) {
        if (parse_simple(text + s, (int)(e - s), out)) return true;
        if (parse_pyfloat(text + s, (int)(e - s), out)) return true;
    }
    // failed: non-ASCII text is first mapped like CPython, then parsed again
    bool ascii = true;
    for (int64_t p = a; p < b; ++p) ascii &= (uint8_t)text[p] < 0x80;
    if (ascii || scratch == nullptr) return false;
    return parse_field_unicode(text, a, b, scratch, out);
}

}  // namespace sa
