// sa_dataset.cuh -- dataset files (CSV rows / TS) parsed and formatted on the
// device: the reference's parse_dataset / format_dataset (datafiles.py:70-143)
// with the same results and the same first error.  Included by sa_kernels.cu
// after the host helpers (fail, SA_CUDA, ensure_device, g_launches).
//
// parse (text bytes resident in HBM):
//   seg_count / seg_write   line breaks of str.splitlines() (\n \r \r\n \v \f
//                           \x1c-\x1e U+0085 U+2028 U+2029), 16 KB per CTA,
//                           plus strict UTF-8 validation (read_dataset decodes
//                           the file as UTF-8, datafiles.py:120-121)
//   line_kernel             warp per line: str.strip() bounds, '@' test, the
//                           last ':' (rsplit, :95), comma counts, label bounds
//   plan / check kernels    format detection (first non-blank line, :75),
//                           header / data roles, field counts, the per-line
//                           errors of :86-110 as an atomicMin over line number
//   field_kernel            warp per data line: every field's byte range
//   parse_kernel            thread per field: float(field) (sa_text.cuh),
//                           first failing field by atomicMin of its global index
//   gather_kernel           labels / header lines joined with '\n'
// format:
//   row_size_kernel         warp per row: bytes of ",".join(repr(v)) [+ ":" label] "\n"
//   row_write_kernel        warp per row: the same text at the row's offset
#pragma once

namespace sa_ds {

using sa::parse_field;
using sa::repr_format;

constexpr int kSegThreads = 256;
constexpr int kSegBytesPerThread = 64;
constexpr int64_t kSegChunk = (int64_t)kSegThreads * kSegBytesPerThread;  // 16 KB
constexpr int64_t kNone = INT64_MAX;

struct Stat {
    unsigned long long nbreaks;
    unsigned long long first_nonblank;
    unsigned long long first_data;
    unsigned long long err_key;     // (line << 2) | kind of the first structural error
    unsigned long long bad_field;   // global index of the first field float() rejects
    unsigned long long bad_utf8;    // first invalid byte
    unsigned long long n_headers;
    unsigned long long nslow;       // fields the fast path left to slow_parse_kernel
    unsigned int nonascii;
    unsigned int ends_with_break;
    unsigned int nonfinite;
    unsigned int format;            // resolved by plan_kernel: 0 csv, 1 ts
};

enum : int { kErrHeader = 0, kErrMissingLabel = 1, kErrRagged = 2 };

// line flags
enum : uint8_t { kNonBlank = 1, kAt = 2, kData = 4, kHeader = 8 };

__device__ __forceinline__ uint8_t byte_at(const char* t, int64_t p) { return (uint8_t)t[p]; }

// Length of the str.splitlines() break starting at byte p (0 if none).
__device__ __forceinline__ int break_len(const char* t, int64_t p, int64_t nb) {
    const uint8_t c = byte_at(t, p);
    if (c == '\n') return (p > 0 && byte_at(t, p - 1) == '\r') ? 0 : 1;
    if (c == '\r') return (p + 1 < nb && byte_at(t, p + 1) == '\n') ? 2 : 1;
    if (c == 0x0b || c == 0x0c || c == 0x1c || c == 0x1d || c == 0x1e) return 1;
    if (c == 0xc2) return (p + 1 < nb && byte_at(t, p + 1) == 0x85) ? 2 : 0;
    if (c == 0xe2)
        return (p + 2 < nb && byte_at(t, p + 1) == 0x80 && (byte_at(t, p + 2) == 0xa8 || byte_at(t, p + 2) == 0xa9))
                   ? 3
                   : 0;
    return 0;
}

// Strict UTF-8 (what bytes.decode('utf-8') accepts): is byte p valid in place?
__device__ bool utf8_ok_at(const char* t, int64_t p, int64_t nb) {
    const uint8_t c = byte_at(t, p);
    if (c < 0x80) return true;
    if ((c & 0xc0) == 0x80) {  // continuation: covered by a lead at most 3 back
        for (int k = 1; k <= 3 && p - k >= 0; ++k) {
            const uint8_t l = byte_at(t, p - k);
            if ((l & 0xc0) == 0x80) continue;
            const int len = (l >= 0xc2 && l <= 0xdf) ? 2 : (l >= 0xe0 && l <= 0xef) ? 3 : (l >= 0xf0 && l <= 0xf4) ? 4 : 0;
            return len > k;
        }
        return false;
    }
    int len;
    uint8_t lo = 0x80, hi = 0xbf;
    if (c >= 0xc2 && c <= 0xdf) len = 2;
    else if (c >= 0xe0 && c <= 0xef) {
        len = 3;
        if (c == 0xe0) lo = 0xa0;
        if (c == 0xed) hi = 0x9f;
    } else if (c >= 0xf0 && c <= 0xf4) {
        len = 4;
        if (c == 0xf0) lo = 0x90;
        if (c == 0xf4) hi = 0x8f;
    } else return false;
    if (p + len > nb) return false;
    const uint8_t c1 = byte_at(t, p + 1);
    if (c1 < lo || c1 > hi) return false;
    for (int k = 2; k < len; ++k)
        if ((byte_at(t, p + k) & 0xc0) != 0x80) return false;
    return true;
}

// any byte < 0x20 or >= 0x80 in a 4-byte word
__device__ __forceinline__ bool word_special(uint32_t w) { return (__vcmpltu4(w, 0x20202020u) | (w & 0x80808080u)) != 0; }

// 16 bytes at w (16-aligned offset); bytes at or past nb read as 0
__device__ __forceinline__ uint4 load16(const char* t, int64_t w, int64_t nb) {
    if (w + 16 <= nb) return *reinterpret_cast<const uint4*>(t + w);
    uint32_t x[4] = {0, 0, 0, 0};
    for (int i = 0; i < 16 && w + i < nb; ++i) x[i >> 2] |= (uint32_t)byte_at(t, w + i) << (8 * (i & 3));
    return make_uint4(x[0], x[1], x[2], x[3]);
}

// bit i set where byte i of the 16-byte word equals c
__device__ __forceinline__ uint32_t match16(uint4 w, uint32_t c4) {
    uint32_t m = 0;
    const uint32_t v[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t e = __vcmpeq4(v[k], c4) & 0x01010101u;  // 1 per matching byte
        m |= ((e * 0x10204080u) >> 28) << (4 * k);           // gather 4 bits
    }
    return m;
}

// bits i with lo <= base + i < hi
__device__ __forceinline__ uint32_t range16(int64_t base, int64_t lo, int64_t hi) {
    const int64_t a = lo - base < 0 ? 0 : (lo - base > 16 ? 16 : lo - base);
    const int64_t b = hi - base < 0 ? 0 : (hi - base > 16 ? 16 : hi - base);
    return (uint32_t)(((1u << b) - 1) & ~((1u << a) - 1)) & 0xffffu;
}

// ---------------------------------------------------------------- segmentation
__device__ __forceinline__ int thread_breaks(const char* t, int64_t nb, int64_t a, int64_t b, bool validate,
                                             Stat* st, int64_t* bstart, int64_t* bnext, int64_t at) {
    int cnt = 0;
    // 16-byte fast path: words without control or non-ASCII bytes hold no
    // break (thread ranges are 64-byte aligned offsets; the host passes a
    // 16-byte aligned text or the bytewise path is taken)
    const bool aligned = ((uintptr_t)t & 15) == 0;
    for (int64_t q = a; q < b; q += 16) {
        bool special = true;
        if (aligned && q + 16 <= b) {
            const uint4 w = *reinterpret_cast<const uint4*>(t + q);
            special = word_special(w.x) || word_special(w.y) || word_special(w.z) || word_special(w.w);
        }
        if (!special) continue;
        const int64_t qe = q + 16 < b ? q + 16 : b;
        for (int64_t p = q; p < qe; ++p) {
            const uint8_t c = byte_at(t, p);
            if (c >= 0x20 && c < 0x80) continue;
            if (c >= 0x80) {
                st->nonascii = 1;  // benign race: every writer stores 1
                if (validate && !utf8_ok_at(t, p, nb)) atomicMin(&st->bad_utf8, (unsigned long long)p);
            }
            const int L = break_len(t, p, nb);
            if (L) {
                if (bstart) {
                    bstart[at + cnt] = p;
                    bnext[at + cnt] = p + L;
                }
                ++cnt;
                if (p + L == nb) st->ends_with_break = 1;
            }
        }
    }
    return cnt;
}

__global__ void __launch_bounds__(kSegThreads) seg_count_kernel(const char* __restrict__ t, int64_t nb, int validate,
                                                                int64_t* counts, Stat* st) {
    const int64_t a0 = blockIdx.x * kSegChunk + (int64_t)threadIdx.x * kSegBytesPerThread;
    const int64_t a = a0 < nb ? a0 : nb, b = a0 + kSegBytesPerThread < nb ? a0 + kSegBytesPerThread : nb;
    int cnt = thread_breaks(t, nb, a, b, validate != 0, st, nullptr, nullptr, 0);
    __shared__ int red[kSegThreads / 32];
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t s = 0;
        for (int k = 0; k < kSegThreads / 32; ++k) s += red[k];
        counts[blockIdx.x] = s;
    }
}

__global__ void __launch_bounds__(kSegThreads) seg_write_kernel(const char* __restrict__ t, int64_t nb,
                                                                const int64_t* __restrict__ chunk_off, int64_t* bstart,
                                                                int64_t* bnext, Stat* st) {
    const int64_t a0 = blockIdx.x * kSegChunk + (int64_t)threadIdx.x * kSegBytesPerThread;
    const int64_t a = a0 < nb ? a0 : nb, b = a0 + kSegBytesPerThread < nb ? a0 + kSegBytesPerThread : nb;
    // count, block exclusive scan, then write in order
    Stat dummy;
    int cnt = thread_breaks(t, nb, a, b, false, &dummy, nullptr, nullptr, 0);
    __shared__ int wsum[kSegThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = cnt;
    for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    int base = 0;
    for (int k = 0; k < wid; ++k) base += wsum[k];
    const int64_t at = chunk_off[blockIdx.x] + base + incl - cnt;
    if (cnt) thread_breaks(t, nb, a, b, false, &dummy, bstart, bnext, at);
    (void)st;
}

// ---------------------------------------------------------------- small scans
// exclusive prefix sum of n int64 (out may alias in); total -> *total
constexpr int kScanTile = 1024;
__global__ void __launch_bounds__(kScanTile) scan_tiles_kernel(const int64_t* in, int64_t n, int64_t* tile_sum) {
    const int64_t i = blockIdx.x * (int64_t)kScanTile + threadIdx.x;
    int64_t v = i < n ? in[i] : 0;
    __shared__ int64_t red[32];
    for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        int64_t s = red[threadIdx.x];
        for (int d = 16; d; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
        if (threadIdx.x == 0) tile_sum[blockIdx.x] = s;
    }
}

__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* total) {
    __shared__ int64_t ws[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t incl = v;
    for (int d = 1; d < 32; d <<= 1) {
        const int64_t u = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += u;
    }
    __syncthreads();
    if (lane == 31) ws[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        int64_t x = lane < nw ? ws[lane] : 0;
        for (int d = 1; d < 32; d <<= 1) {
            const int64_t u = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += u;
        }
        if (lane < nw) ws[lane] = x;  // inclusive per warp
    }
    __syncthreads();
    const int64_t before = wid ? ws[wid - 1] : 0;
    *total = ws[((blockDim.x + 31) >> 5) - 1];
    return before + incl - v;
}

__global__ void __launch_bounds__(kScanTile) scan_partials_kernel(int64_t* tile_sum, int64_t ntiles, int64_t* total) {
    int64_t carry = 0;
    for (int64_t base = 0; base < ntiles; base += kScanTile) {
        const int64_t i = base + threadIdx.x;
        const int64_t v = i < ntiles ? tile_sum[i] : 0;
        int64_t tot;
        const int64_t ex = block_excl_scan(v, &tot);
        if (i < ntiles) tile_sum[i] = carry + ex;
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(kScanTile) scan_apply_kernel(const int64_t* in, int64_t n, const int64_t* tile_off,
                                                               int64_t* out) {
    const int64_t i = blockIdx.x * (int64_t)kScanTile + threadIdx.x;
    const int64_t v = i < n ? in[i] : 0;
    int64_t tot;
    const int64_t ex = block_excl_scan(v, &tot);
    if (i < n) out[i] = tile_off[blockIdx.x] + ex;
}

// ---------------------------------------------------------------- lines
struct Lines {
    int64_t n;
    const int64_t* bstart;  // break k starts at bstart[k] (line k ends there)
    const int64_t* bnext;   // line k+1 starts at bnext[k]
    int64_t nbreaks;
    int64_t* s;      // stripped bounds
    int64_t* e;
    int64_t* colon;  // last ':' in [s, e), -1 if none
    int64_t* ncomma_all;
    int64_t* ncomma_vals;  // commas in [s, colon)
    int64_t* lab_s;  // stripped label bounds (after the colon)
    int64_t* lab_e;
    uint8_t* flags;
};

// Unicode whitespace (str.isspace) sequence length starting at byte p, or 0.
__device__ __forceinline__ int ws_len(const char* t, int64_t p, int64_t end) {
    const uint8_t c = byte_at(t, p);
    if (c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f)) return 1;
    if (c < 0xc2) return 0;
    uint32_t cp;
    const int k = sa::utf8_decode(t, p, end, &cp);
    return sa::is_unicode_space(cp) ? k : 0;
}

__device__ __forceinline__ bool is_cont(const char* t, int64_t p) { return (byte_at(t, p) & 0xc0) == 0x80; }

// is the character starting at p (a lead byte) a non-whitespace char?
__device__ __forceinline__ bool nonws_char_at(const char* t, int64_t p, int64_t end) {
    return !is_cont(t, p) && ws_len(t, p, end) == 0;
}

// str.strip() of [a, b) by one thread (labels: short)
__device__ void strip_serial(const char* t, int64_t* pa, int64_t* pb) {
    int64_t a = *pa, b = *pb;
    while (a < b) {
        const int k = ws_len(t, a, b);
        if (!k) break;
        a += k;
    }
    while (b > a) {
        int64_t q = b - 1;
        while (q > a && is_cont(t, q)) --q;
        if (ws_len(t, q, b) != (int)(b - q)) break;
        b = q;
    }
    *pa = a;
    *pb = b;
}

__device__ __forceinline__ bool ascii_graph(uint8_t c) { return c > 0x20 && c < 0x7f; }

__global__ void __launch_bounds__(256) line_kernel(const char* __restrict__ t, int64_t nb, Lines L, Stat* st) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const bool aligned = ((uintptr_t)t & 15) == 0;
    for (int64_t k = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); k < L.n; k += nw) {
        const int64_t a = k == 0 ? 0 : L.bnext[k - 1];
        const int64_t b = k < L.nbreaks ? L.bstart[k] : nb;
        // str.strip(): the common line starts and ends with a printable ASCII byte
        int64_t s = b;
        if (a < b && ascii_graph(byte_at(t, a))) {
            s = a;
        } else {
            for (int64_t p0 = a; p0 < b; p0 += 32) {
                const int64_t p = p0 + lane;
                const unsigned m = __ballot_sync(0xffffffffu, p < b && nonws_char_at(t, p, b));
                if (m) {
                    s = p0 + __ffs(m) - 1;
                    break;
                }
            }
        }
        int64_t e = s;
        if (s < b && ascii_graph(byte_at(t, b - 1))) {
            e = b;
        } else {
            for (int64_t p1 = b; p1 > s; p1 -= 32) {
                const int64_t p = p1 - 1 - lane;
                const unsigned m = __ballot_sync(0xffffffffu, p >= s && nonws_char_at(t, p, b));
                if (m) {
                    const int64_t q = p1 - 1 - (__ffs(m) - 1);  // lowest lane = highest position
                    uint32_t cp;
                    e = q + sa::utf8_decode(t, q, b, &cp);
                    break;
                }
            }
        }
        // last ':' in [s, e) (labels are short: found in the first step)
        int64_t colon = -1;
        for (int64_t p1 = e; p1 > s; p1 -= 32) {
            const int64_t p = p1 - 1 - lane;
            const unsigned m = __ballot_sync(0xffffffffu, p >= s && t[p] == ':');
            if (m) {
                colon = p1 - 1 - (__ffs(m) - 1);
                break;
            }
        }
        // commas in [s, e) and in [s, colon): 16 bytes per lane per step
        int64_t call = 0, cval = 0;
        if (aligned) {
            for (int64_t w = (s & ~(int64_t)15) + 16 * lane; w < e; w += 512) {
                const uint32_t m = match16(load16(t, w, nb), 0x2c2c2c2cu);
                call += __popc(m & range16(w, s, e));
                cval += __popc(m & range16(w, s, colon));
            }
        } else {
            for (int64_t p = s + lane; p < e; p += 32) {
                const bool c = t[p] == ',';
                call += c;
                cval += c && p < colon;
            }
        }
        for (int d = 16; d; d >>= 1) {
            call += __shfl_xor_sync(0xffffffffu, call, d);
            cval += __shfl_xor_sync(0xffffffffu, cval, d);
        }
        if (lane == 0) {
            uint8_t f = 0;
            if (e > s) {
                f |= kNonBlank;
                if (t[s] == '@') f |= kAt;
                atomicMin(&st->first_nonblank, (unsigned long long)k);
            }
            L.s[k] = s;
            L.e[k] = e;
            L.colon[k] = colon;
            L.ncomma_all[k] = call;
            L.ncomma_vals[k] = cval;
            int64_t ls = colon >= 0 ? colon + 1 : e, le = e;
            strip_serial(t, &ls, &le);
            L.lab_s[k] = ls;
            L.lab_e[k] = le;
            L.flags[k] = f;
        }
    }
}

// roles and field counts; fmt < 0: detect from the first non-blank line
__global__ void plan_kernel(Lines L, int fmt, int64_t* nfields, int64_t* is_data, int64_t* is_header,
                            int64_t* hdr_bytes, int64_t* lab_bytes, Stat* st) {
    const int ts = fmt >= 0 ? fmt : (st->first_nonblank != (unsigned long long)kNone &&
                                     (L.flags[st->first_nonblank] & kAt) ? 1 : 0);
    if (blockIdx.x == 0 && threadIdx.x == 0) st->format = ts;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < L.n; k += (int64_t)gridDim.x * blockDim.x) {
        uint8_t f = L.flags[k];
        int64_t nf = 0, d = 0, h = 0;
        if (f & kNonBlank) {
            if (ts && (f & kAt)) {
                h = 1;
                f |= kHeader;
            } else {
                d = 1;
                f |= kData;
                nf = ts ? (L.colon[k] >= 0 ? L.ncomma_vals[k] + 1 : 0) : L.ncomma_all[k] + 1;
                atomicMin(&st->first_data, (unsigned long long)k);
            }
        }
        L.flags[k] = f;
        nfields[k] = nf;
        is_data[k] = d;
        is_header[k] = h;
        hdr_bytes[k] = h ? L.e[k] - L.s[k] + 1 : 0;
        lab_bytes[k] = (d && ts) ? L.lab_e[k] - L.lab_s[k] + 1 : 0;
    }
}

__global__ void check_kernel(Lines L, const int64_t* nfields, Stat* st) {
    const unsigned long long fd = st->first_data;
    const int ts = (int)st->format;
    const int64_t w = fd != (unsigned long long)kNone ? nfields[fd] : 0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < L.n; k += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t f = L.flags[k];
        int err = -1;
        if ((f & kHeader) && fd != (unsigned long long)kNone && (unsigned long long)k > fd) err = kErrHeader;
        if (f & kData) {
            if (ts && L.colon[k] < 0) err = kErrMissingLabel;
            else if (nfields[k] != w) err = kErrRagged;
        }
        if (err >= 0) atomicMin(&st->err_key, ((unsigned long long)k << 2) | (unsigned)err);
    }
}

// field byte ranges of every data line with k <= last_line
__global__ void __launch_bounds__(256) field_kernel(const char* __restrict__ t, Lines L, const int64_t* nfields,
                                                   const int64_t* field_off, int64_t last_line, int64_t* fs,
                                                   int64_t* fe, const Stat* st) {
    const bool ts = st->format != 0;
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t nl = last_line + 1 < L.n ? last_line + 1 : L.n;
    for (int64_t k = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); k < nl; k += nw) {
        const int64_t nf = nfields[k];
        if (nf == 0) continue;
        const int64_t s = L.s[k];
        const int64_t vend = ts ? L.colon[k] : L.e[k];  // values part (rsplit(':', 1), :95)
        const int64_t base = field_off[k];
        int64_t idx = 0;  // fields started so far
        if (lane == 0) fs[base] = s;
        for (int64_t p0 = s; p0 < vend; p0 += 32) {
            const int64_t p = p0 + lane;
            const bool c = p < vend && t[p] == ',';
            const unsigned m = __ballot_sync(0xffffffffu, c);
            if (c) {
                const int64_t j = idx + __popc(m & ((1u << lane) - 1));  // comma j ends field j
                fe[base + j] = p;
                fs[base + j + 1] = p + 1;
            }
            idx += __popc(m);
        }
        if (lane == 0) fe[base + nf - 1] = vend;
    }
}

__global__ void __launch_bounds__(256) parse_kernel(const char* __restrict__ t, const int64_t* __restrict__ fs,
                                                   const int64_t* __restrict__ fe, int64_t nf, char* scratch,
                                                   double* __restrict__ out, Stat* st) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nf; i += (int64_t)gridDim.x * blockDim.x) {
        double v = 0.0;
        if (!parse_field(t, fs[i], fe[i], scratch, &v)) atomicMin(&st->bad_field, (unsigned long long)i);
        const uint64_t bits = (uint64_t)__double_as_longlong(v);
        if ((bits & 0x7ff0000000000000ull) == 0x7ff0000000000000ull) st->nonfinite = 1;
        out[i] = v;
    }
}

// Fused field split + float(): warp per data line, the line streamed
// through shared memory in 1 KB windows (coalesced 16-byte loads); commas
// found with byte-compare masks and a warp prefix count; each lane parses
// whole fields out of shared memory and the row's values are stored
// coalesced at field_off[k] + j (the batch is row-major n x width).
constexpr int kParseWarps = 8;
constexpr int kWin = 1024;

struct SlowField {
    int64_t gi, a, b;  // global field index, byte range
};

__device__ __forceinline__ void put_value(int64_t gi, const char* t, int64_t fa, int64_t fb, bool ok, double v,
                                          double* out, Stat* st, SlowField* slow, int64_t slow_cap) {
    if (!ok) {  // left for slow_parse_kernel (full grammar, exact rounding, Unicode, errors)
        const unsigned long long q = atomicAdd(&st->nslow, 1ull);
        if ((int64_t)q < slow_cap) slow[q] = SlowField{gi, fa, fb};
        return;
    }
    if (((uint64_t)__double_as_longlong(v) & 0x7ff0000000000000ull) == 0x7ff0000000000000ull) st->nonfinite = 1;
    out[gi] = v;
}

// field text without surrounding ASCII whitespace, fast path only
__device__ __forceinline__ bool parse_fast(const char* t, int64_t a, int64_t b, double* v) {
    while (a < b && sa::py_isspace(t[a])) ++a;
    while (b > a && sa::py_isspace(t[b - 1])) --b;
    return b - a <= 64 && sa::parse_simple(t + a, (int)(b - a), v);
}

__global__ void __launch_bounds__(kParseWarps * 32) rows_parse_kernel(const char* __restrict__ t, int64_t nb, Lines L,
                                                                      const int64_t* __restrict__ nfields,
                                                                      const int64_t* __restrict__ field_off,
                                                                      double* __restrict__ out, Stat* st,
                                                                      SlowField* slow, int64_t slow_cap) {
    __shared__ __align__(16) char win[kParseWarps][kWin];
    __shared__ uint16_t cpos[kParseWarps][kWin];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    char* buf = win[wid];
    uint16_t* cp = cpos[wid];
    const bool ts = st->format != 0;
    const int64_t nwarps = (int64_t)gridDim.x * kParseWarps;
    for (int64_t k = blockIdx.x * (int64_t)kParseWarps + wid; k < L.n; k += nwarps) {
        const int64_t nf = nfields[k];
        if (nf == 0) continue;
        const int64_t s = L.s[k];
        const int64_t vend = ts ? L.colon[k] : L.e[k];
        const int64_t base = field_off[k];
        int64_t fstart = s;  // start of the field in progress
        int64_t j = 0;       // fields completed
        for (int64_t w0 = s & ~(int64_t)15; w0 < vend; w0 += kWin) {
            // stage [w0, w0 + kWin) and mark commas; lane covers 32 contiguous bytes
            const int64_t wa = w0 + 32 * lane;
            const uint4 v0 = load16(t, wa, nb), v1 = load16(t, wa + 16, nb);
            *reinterpret_cast<uint4*>(buf + 32 * lane) = v0;
            *reinterpret_cast<uint4*>(buf + 32 * lane + 16) = v1;
            const uint32_t m = (match16(v0, 0x2c2c2c2cu) & range16(wa, s, vend)) |
                               ((match16(v1, 0x2c2c2c2cu) & range16(wa + 16, s, vend)) << 16);
            const int c = __popc(m);
            int incl = c;
            for (int d = 1; d < 32; d <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += u;
            }
            int o = incl - c;
            for (uint32_t mm = m; mm; mm &= mm - 1) cp[o++] = (uint16_t)(32 * lane + __ffs(mm) - 1);
            const int ncomma = __shfl_sync(0xffffffffu, incl, 31);
            __syncwarp();
            for (int q = lane; q < ncomma; q += 32) {
                const int64_t fb = w0 + cp[q];
                const int64_t fa = q == 0 ? fstart : w0 + cp[q - 1] + 1;
                double v = 0.0;
                const bool ok = fa >= w0 ? parse_fast(buf - w0, fa, fb, &v) : parse_fast(t, fa, fb, &v);
                put_value(base + j + q, t, fa, fb, ok, v, out, st, slow, slow_cap);
            }
            if (ncomma) fstart = w0 + cp[ncomma - 1] + 1;
            j += ncomma;
            __syncwarp();
        }
        if (lane == 0) {  // the last field ends at the values' end
            double v = 0.0;
            const bool ok = parse_fast(t, fstart, vend, &v);
            put_value(base + nf - 1, t, fstart, vend, ok, v, out, st, slow, slow_cap);
        }
    }
}

// the fields the fast path could not decide: full float() semantics
__global__ void __launch_bounds__(128) slow_parse_kernel(const char* __restrict__ t, const SlowField* __restrict__ slow,
                                                        int64_t n, char* scratch, double* out, Stat* st) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const SlowField f = slow[i];
        double v = 0.0;
        if (!parse_field(t, f.a, f.b, scratch, &v)) atomicMin(&st->bad_field, (unsigned long long)f.gi);
        if (((uint64_t)__double_as_longlong(v) & 0x7ff0000000000000ull) == 0x7ff0000000000000ull) st->nonfinite = 1;
        out[f.gi] = v;
    }
}

// join the selected ranges with a trailing '\n' each at off[k]
__global__ void __launch_bounds__(256) gather_kernel(const char* __restrict__ t, const int64_t* sel, const int64_t* a,
                                                    const int64_t* off, int64_t n, char* out) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t k = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); k < n; k += nw) {
        const int64_t len = sel[k];
        if (len == 0) continue;
        const int64_t src = a[k], dst = off[k];
        for (int64_t q = lane; q < len - 1; q += 32) out[dst + q] = t[src + q];
        if (lane == 0) out[dst + len - 1] = '\n';
    }
}

__global__ void add_kernel(int64_t* x, int64_t n, int64_t v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] += v;
}

// ---------------------------------------------------------------- format
__global__ void __launch_bounds__(256) row_size_kernel(const double* __restrict__ v, int64_t n, int64_t len, int ts,
                                                      const int64_t* __restrict__ lab_off, int64_t* row_bytes) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += nw) {
        int64_t tot = 0;
        for (int64_t j = lane; j < len; j += 32) tot += sa::repr_len(sa::repr_decompose(v[r * len + j]));
        for (int d = 16; d; d >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, d);
        if (lane == 0) {
            tot += len - 1 + 1;  // commas + '\n'
            if (ts) tot += 1 + (lab_off ? lab_off[r + 1] - lab_off[r] : 0);
            row_bytes[r] = tot;
        }
    }
}

// Warp per row: 32 values at a time are rendered into a shared-memory
// staging buffer at their prefix-summed offsets, and full 32-byte runs are
// flushed with coalesced stores (one sector per warp store).
constexpr int kFmtWarps = 8;
constexpr int kStage = 2048;

__device__ __forceinline__ void flush_stage(char* out, int64_t pos, const char* stg, int nbytes, int lane) {
    // byte-coalesced copy; 4-byte stores once the destination is aligned
    int i = 0;
    const int head = (int)((4 - (pos & 3)) & 3) < nbytes ? (int)((4 - (pos & 3)) & 3) : nbytes;
    if (lane < head) out[pos + lane] = stg[lane];
    i = head;
    const int nw = (nbytes - i) >> 2;
    uint32_t* o4 = reinterpret_cast<uint32_t*>(out + pos + i);
    for (int q = lane; q < nw; q += 32) {
        const char* src = stg + i + 4 * q;
        o4[q] = (uint32_t)(uint8_t)src[0] | ((uint32_t)(uint8_t)src[1] << 8) | ((uint32_t)(uint8_t)src[2] << 16) |
                ((uint32_t)(uint8_t)src[3] << 24);
    }
    i += 4 * nw;
    if (lane < nbytes - i) out[pos + i + lane] = stg[i + lane];
}

__global__ void __launch_bounds__(kFmtWarps * 32) row_write_kernel(const double* __restrict__ v, int64_t n, int64_t len,
                                                                  int ts, const char* __restrict__ labels,
                                                                  const int64_t* __restrict__ lab_off,
                                                                  const int64_t* __restrict__ row_off, char* out) {
    __shared__ char stage[kFmtWarps][kStage + 64];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    char* stg = stage[wid];
    const int64_t nw = (int64_t)gridDim.x * kFmtWarps;
    for (int64_t r = blockIdx.x * (int64_t)kFmtWarps + wid; r < n; r += nw) {
        int64_t pos = row_off[r];  // file offset of stg[0]
        int fill = 0;              // bytes staged
        for (int64_t j0 = 0; j0 < len; j0 += 32) {
            const int64_t j = j0 + lane;
            sa::Repr rp;
            int k = 0;
            if (j < len) {
                rp = sa::repr_decompose(v[r * len + j]);
                k = sa::repr_len(rp) + (j + 1 < len ? 1 : 0);
            }
            int incl = k;
            for (int d = 1; d < 32; d <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += u;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            if (fill + total > kStage) {  // at most 32 * 25 bytes per step
                flush_stage(out, pos, stg, fill, lane);
                pos += fill;
                fill = 0;
                __syncwarp();
            }
            if (j < len) {
                char* d = stg + fill + incl - k;
                sa::repr_write(rp, d);
                if (j + 1 < len) d[k - 1] = ',';
            }
            fill += total;
            __syncwarp();
        }
        if (ts) {
            const int64_t la = lab_off ? lab_off[r] : 0, lb = lab_off ? lab_off[r + 1] : 0;
            if (fill + 1 + (lb - la) + 1 > kStage) {
                flush_stage(out, pos, stg, fill, lane);
                pos += fill;
                fill = 0;
                __syncwarp();
            }
            if (fill + 1 + (lb - la) + 1 <= kStage) {
                if (lane == 0) stg[fill] = ':';
                for (int64_t q = lane; q < lb - la; q += 32) stg[fill + 1 + q] = labels[la + q];
                fill += 1 + (int)(lb - la);
            } else {  // a label longer than the stage goes straight out
                if (lane == 0) out[pos] = ':';
                for (int64_t q = lane; q < lb - la; q += 32) out[pos + 1 + q] = labels[la + q];
                pos += 1 + (lb - la);
            }
        }
        if (lane == 0) stg[fill] = '\n';
        ++fill;
        __syncwarp();
        flush_stage(out, pos, stg, fill, lane);
        __syncwarp();
    }
}

}  // namespace sa_ds
