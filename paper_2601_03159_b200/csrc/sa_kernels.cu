// sa_kernels.cu -- the fused augmentation-chain kernel, the spectral
// transform kernels, and the C ABI (include/seriesaug_b200.h).
//
// Execution model: a persistent grid of one-warp CTAs; each
// warp takes series (rows) round-robin.  Per row:
//   1. TMA bulk copy (cp.async.bulk, mbarrier completion) of the input row
//      into shared memory -- one HBM read per series;
//   2. gate pre-pass: lane j derives stage j's Philox key (reference
//      core.py:77-82) and its first Philox block; random() < p of word 0 is
//      the gate (core.py:235).  Words 1..3 stay cached for the stage's first
//      draws;
//   3. every fired stage runs in smem (sa_ops.cuh), per-sample order;
//   4. finiteness is checked after every arithmetic stage (the reference's
//      per-stage Batch() re-validation, core.py:259 -> :104) into a flag;
//   5. coalesced 128-bit stores of the output row -- one HBM write per series.
#include <cuda_runtime.h>
#include <immintrin.h>

#include <algorithm>
#include <initializer_list>
#include <chrono>
#include <cmath>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <thread>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <functional>
#include <vector>

#include "../../include/seriesaug_b200.h"
#include "sa_dtw.cuh"
#include "sa_text.cuh"
#include "sa_dataset.cuh"
#include "sa_ops.cuh"
#include "sa_fft_cta.cuh"

namespace sa {

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
// TMA 1-D bulk copy global -> shared, completion via mbarrier tx count.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Ampere-style async copy of one 8-byte word global -> shared (L2 only);
// used where the source is not a 16-byte-aligned contiguous row (TMA's
// requirement), e.g. interleaving separate re / im arrays.
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// TMA 1-D bulk copy shared -> global (bulk-group completion).  The issuing
// thread waits for the source reads (wait_read) before the buffer is reused.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// ------------------------------------------------------------ smem layout
struct Layout {
    uint32_t buf_a, buf_b, win, scache, small, iscr, bar, total;
};

__host__ __device__ inline uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }

__host__ __device__ inline Layout make_layout(int lcap, int ns, int small_words, int iscr_words) {
    Layout l;
    uint32_t o = 0;
    l.buf_a = o; o = align16(o + 8u * (uint32_t)lcap);
    l.buf_b = o; o = align16(o + 8u * (uint32_t)lcap);
    l.win = o; o = align16(o + 8u * SA_WIN);
    l.scache = o; o = align16(o + 48u * (uint32_t)(ns > 0 ? ns : 1));
    l.small = o; o = align16(o + 8u * (uint32_t)small_words);
    l.iscr = o; o = align16(o + 4u * (uint32_t)iscr_words);
    l.bar = o; o = align16(o + 8u);
    l.total = o;
    return l;
}

// Dynamic shared memory shared by the CTA after the warps' slices: numpy's
// ziggurat fast-path table and the adaptive-lockstep key slots (2 x OR, AND).
constexpr size_t kCtaShared = 256 * sizeof(ZigEntry) + 4 * sizeof(unsigned long long);

// ------------------------------------------------------------ the kernel
// GMEM: the row buffers live in p.gbuf (long series); the shared-memory
// instantiation keeps them provably in shared memory (LDS/STS, not generic
// accesses) -- the two are separate kernels for that reason.
// MAXT: threads per CTA the register allocation targets -- 384 (12 warps,
// 168 registers) for the general kernel; the short-series instantiation
// (chain_kernel<false, kWideThreads>) trades registers for more series in
// flight, since short rows are latency bound on per-row fixed costs.
#ifndef SA_WIDE_THREADS
#define SA_WIDE_THREADS 512
#endif
constexpr int kWideThreads = SA_WIDE_THREADS;
// ODD: spectral stages whose FFT plan is not plain radix-8/4/2 (generic
// odd-prime passes, Bluestein, the odd-length real transforms of sa_fft.cuh);
// separate instantiations, so the kernel the power-of-two lengths run is
// generated without that code (measured: inlining the odd-length transform
// alone cost config 5 1%).
template <bool GMEM, int MAXT = 384, bool ODD = false>
__global__ void __launch_bounds__(MAXT) chain_kernel(const __grid_constant__ ChainParams p) {
    extern __shared__ __align__(16) unsigned char smem_all[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    // the two row buffers sit in this warp's shared-memory slice, or -- for
    // series too long for it -- in the warp's slot of a global scratch
    const Layout lay = make_layout(GMEM ? 0 : p.lcap, p.ns, p.small_words, p.iscr_words);
    unsigned char* smem = smem_all + (size_t)wid * lay.total;  // this warp's slice
    double* A = GMEM ? p.gbuf + ((int64_t)blockIdx.x * nw + wid) * 2 * (int64_t)p.lcap
                     : reinterpret_cast<double*>(smem + lay.buf_a);
    double* B = GMEM ? A + p.lcap : reinterpret_cast<double*>(smem + lay.buf_b);
    uint64_t* scache = reinterpret_cast<uint64_t*>(smem + lay.scache);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + lay.bar);
    Warp w;
    w.lane = lane;
    w.win = reinterpret_cast<uint64_t*>(smem + lay.win);
    w.small = reinterpret_cast<double*>(smem + lay.small);
    w.iscr = reinterpret_cast<int32_t*>(smem + lay.iscr);
    w.lcap = p.lcap;
    ZigEntry* zs = reinterpret_cast<ZigEntry*>(smem_all + (size_t)nw * lay.total);  // CTA-shared
    for (int i = threadIdx.x; i < 256; i += blockDim.x) zs[i] = g_zig[i];
    w.zig = zs;
    __syncthreads();

    if (lane == 0) mbar_init(bar, 1);
    __syncwarp();
    // adaptive lockstep: OR / AND of the rows' gate keys per row iteration
    // (double-buffered by iteration parity).  One group: the whole CTA
    // (lockstep groups smaller than the CTA multiply the instruction working
    // set -- measured 1.6-2.8x slower).
    unsigned long long* s_kor = reinterpret_cast<unsigned long long*>(zs + 256);
    unsigned long long* s_kand = s_kor + 2;
    if (threadIdx.x < 2) {
        s_kor[threadIdx.x] = 0ull;
        s_kand[threadIdx.x] = ~0ull;
    }
    __syncthreads();
    int it = 0;
    bool pend_store = false;  // a bulk store of this warp's row is in flight
    uint32_t phase = 0;
    uint32_t flags = 0;
    const int r = p.repeat_r;
    const uint32_t in_bytes = 8u * (uint32_t)p.len_in;

    // Rows are dealt to warps; the trip count is uniform across the CTA so
    // the stage-boundary barriers below are reached by every warp.
    for (int64_t base = (int64_t)blockIdx.x * nw; base < p.rows_out; base += (int64_t)gridDim.x * nw) {
        const int64_t slot = base + wid;
        const bool active = slot < p.rows_out;
        const int64_t row = (active && p.order) ? (int64_t)p.order[slot] : slot;
        const int64_t in_row = (active ? row : 0) / r;
        const double* src = p.in + in_row * (int64_t)p.len_in;
        uint64_t fire_lo = 0;  // fire bits of stages 0..63
        if (!GMEM && pend_store) {  // the previous row's bulk store has read its buffer
            if (lane == 0) bulk_wait_read();
            pend_store = false;
            __syncwarp();
        }
        if (active) {
        // 1. stage the input row
        if (p.bulk_in) {
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(bar, in_bytes);
                bulk_g2s(A, src, in_bytes, bar);
            }
        } else {
            for (int t = lane; t < p.len_in; t += 32) A[t] = __ldcs(&src[t]);  // streaming: keep L2 for the row scratch
        }
        // 2. gate pre-pass (overlaps the bulk copy)
        for (int j0 = 0; j0 < p.ns; j0 += 32) {
            const int j = j0 + lane;
            bool fire = false;
            if (j < p.ns) {
                const DevStage& st = p.st[j];
                const uint64_t series =
                    st.post_repeat ? (uint64_t)(p.offset * r + row) : (uint64_t)(p.offset + in_row);
                uint64_t k0, k1, o0, o1, o2, o3;
                derive_key(p.seed, (uint64_t)st.index, series, k0, k1);
                philox(k0, k1, 1, o0, o1, o2, o3);
                uint64_t* c = scache + 6 * j;
                c[0] = k0; c[1] = k1; c[2] = o0; c[3] = o1; c[4] = o2; c[5] = o3;
                fire = u53(o0) < st.prob && st.op != SA_OP_REPEAT;
            }
            fire_lo |= (uint64_t)__ballot_sync(SA_FULL, fire) << j0;
        }
        if (p.bulk_in) {
            mbar_wait(bar, phase);
            phase ^= 1u;
        }
        __syncwarp();
        // input finiteness (Batch invariant, core.py:104)
        {
            Finite bad;
#pragma unroll 4
            for (int t = lane; t < p.len_in; t += 32) bad.chk(A[t]);
            if (__any_sync(SA_FULL, bad.any())) flags |= SA_FLAG_NONFINITE;
        }
        }
        // 3. the chain (stage-major across the CTA when sync_every > 0).  When
        // every row of the CTA fires the same gated stages (uni_mask bits) the
        // warps do the same work and stay together without the in-row
        // barriers; one barrier per row iteration re-aligns them.
        bool uniform = false;
        if (p.sync_every) {
            const int b = it & 1;
            if (lane == 0 && active) {
                atomicOr(&s_kor[b], (unsigned long long)(fire_lo & p.uni_mask));
                atomicAnd(&s_kand[b], (unsigned long long)(fire_lo & p.uni_mask));
            }
            if (threadIdx.x == 0) {  // reset the other parity's slots for the next iteration
                s_kor[b ^ 1] = 0ull;
                s_kand[b ^ 1] = ~0ull;
            }
            __syncthreads();
            uniform = p.uni_mask != ~0ull && (s_kor[b] & ~s_kand[b]) == 0ull;
            ++it;
        }
        Finite bad;  // per-lane: some stage output was non-finite
        double* cur = A;
        double* oth = B;
        int L = p.len_in;
        double2* held = nullptr;  // the row's half spectrum between fused spectral stages
        for (int j = 0; j < p.ns; ++j) {
            if (!uniform && j && ((p.sync_mask >> j) & 1ull)) __syncthreads();  // j = 0: the check above
            if (!active || !((fire_lo >> j) & 1ull)) continue;
            const DevStage& st = p.st[j];
            const uint64_t* c = scache + 6 * j;
            WStream s;
            s.k0 = c[0];
            s.k1 = c[1];
            s.win = c + 2;
            s.winbuf = w.win;
            s.wb = 0;
            s.wn = 4;
            s.wpos = 1;  // word 0 was the gate
            s.has32 = 0;
            s.u32 = 0;
            bool arith = false;
            switch (st.op) {
                case SA_OP_JITTER:
                case SA_OP_NOISE_GAUSSIAN: arith = op_gauss(st, s, cur, oth, L, w, bad); break;
                case SA_OP_SCALE: arith = op_scale(st, s, cur, oth, L, w, bad); break;
                case SA_OP_ROTATE: arith = op_rotate(cur, L, w); break;
                case SA_OP_PERMUTE: arith = op_permute(st, s, cur, oth, L, w); break;
                case SA_OP_CROP: arith = op_crop(st, s, cur, oth, L, w); break;
                case SA_OP_REVERSE: arith = op_reverse(cur, oth, L, w); break;
                case SA_OP_RESIZE: arith = op_resize(st, cur, oth, L, w, bad); break;
                case SA_OP_QUANTIZE: arith = op_quantize(st, cur, L, w, bad); break;
                case SA_OP_DRIFT: arith = op_drift(st, s, cur, oth, L, w, bad); break;
                case SA_OP_NOISE_UNIFORM: arith = op_uniform(st, s, cur, L, w, bad); break;
                case SA_OP_NOISE_SPIKE: arith = op_spike(st, s, cur, oth, L, w, bad); break;
                case SA_OP_NOISE_SLOPE: arith = op_slope(st, s, cur, L, w, bad); break;
                case SA_OP_APP:
                case SA_OP_FREQ_MASK:
                case SA_OP_SINUSOID: {
                    // Consecutive spectral stages share one spectrum: the
                    // reference's irfft -> rfft between them is the identity
                    // up to rounding once DC (and Nyquist) imaginary parts
                    // are re-pinned to 0 (freqaugment.py:40-45), so the row
                    // stays in the frequency domain until the last one.
                    const uint64_t later = (j + 1 < 64) ? (fire_lo >> (j + 1)) : 0;
                    const int nx = later ? j + 1 + __ffsll((long long)later) - 1 : p.ns;
                    const bool keep = nx < p.ns && is_spectral_op(p.st[nx].op) && !spectral_noop(p.st[nx]);
                    arith = op_spectral<ODD>(st, s, cur, oth, L, w, held, keep, bad);
                    break;
                }
                case SA_OP_TIME_WARP: arith = op_time_warp(st, s, cur, oth, L, w, flags, bad); break;
                case SA_OP_WINDOW_WARP: arith = op_window_warp(st, s, cur, oth, L, w, flags, bad); break;
                case SA_OP_DROPOUT: arith = op_dropout(st, s, cur, L, w); break;
                case SA_OP_POOL: arith = op_pool(st, cur, L, w, bad); break;
                case SA_OP_CONVOLVE: arith = op_convolve(st, p.aux, cur, oth, L, w, bad); break;
                case SA_OP_SPEED_WARP: arith = op_speed_warp(st, s, cur, oth, L, w, bad); break;
                default: break;
            }
            if (arith) {  // ops that do not fold the check into their writes
#pragma unroll 4
                for (int t = lane; t < L; t += 32) bad.chk(cur[t]);
            }
        }
        if (__any_sync(SA_FULL, bad.any())) flags |= SA_FLAG_NONFINITE;
        // 5. write the row
        if (!active) continue;
        double* dst = p.out + row * (int64_t)p.len_out;
        if (!GMEM && (p.len_out & 1) == 0 && ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0)) {
            // one TMA bulk store of the row: the generic-proxy writes are made
            // visible to the async proxy, then lane 0 issues it
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) bulk_s2g(dst, cur, 8u * (uint32_t)p.len_out);
            pend_store = true;
            continue;
        }
        if ((p.len_out & 1) == 0 && ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0)) {
            const double2* c2 = reinterpret_cast<const double2*>(cur);
            double2* d2 = reinterpret_cast<double2*>(dst);
            for (int t = lane; t < p.len_out / 2; t += 32) __stcs(&d2[t], c2[t]);
        } else {
            for (int t = lane; t < p.len_out; t += 32) __stcs(&dst[t], cur[t]);
        }
        __syncwarp();
    }
    if (!GMEM && pend_store && lane == 0) bulk_wait_all();
    if (flags && lane == 0) atomicOr(p.flags, flags);
}


// ------------------------------------------------------------ fire-pattern scheduling
// The stage barrier makes every stage cost the slowest firing warp of the
// CTA.  Rows whose gates fire the same expensive stages are therefore
// grouped: key = fire bits of the (up to 16) most expensive gated stages,
// counting-sorted; the chain kernel takes rows in that order.  Output rows
// are still written to their own positions, so results are unchanged.
__device__ __forceinline__ uint32_t fire_key(const ChainParams& p, int64_t row) {
    const int64_t in_row = row / p.repeat_r;
    uint32_t key = 0;
    for (int q = 0; q < p.key_bits; ++q) {
        const DevStage& st = p.st[p.key_stage[q]];
        const uint64_t series =
            st.post_repeat ? (uint64_t)(p.offset * p.repeat_r + row) : (uint64_t)(p.offset + in_row);
        uint64_t k0, k1, o0, o1, o2, o3;
        derive_key(p.seed, (uint64_t)st.index, series, k0, k1);
        philox(k0, k1, 1, o0, o1, o2, o3);
        key = (key << 1) | (u53(o0) < st.prob ? 1u : 0u);
    }
    return key;
}

__global__ void __launch_bounds__(256) key_hist_kernel(const __grid_constant__ ChainParams p, uint32_t* keys,
                                                       uint32_t* hist) {
    for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < p.rows_out;
         row += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = fire_key(p, row);
        keys[row] = k;
        atomicAdd(&hist[k], 1u);
    }
}

// exclusive scan of nb <= 65536 counters, one CTA of 1024 threads
__global__ void __launch_bounds__(1024) key_scan_kernel(uint32_t* hist, int nb) {
    __shared__ uint32_t part[1024];
    const int per = (nb + 1023) / 1024;
    const int a = threadIdx.x * per, b = min(nb, a + per);
    uint32_t s = 0;
    for (int i = a; i < b; ++i) s += hist[i];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        uint32_t v = threadIdx.x >= off ? part[threadIdx.x - off] : 0u;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    uint32_t run = threadIdx.x ? part[threadIdx.x - 1] : 0u;
    for (int i = a; i < b; ++i) {
        const uint32_t c = hist[i];
        hist[i] = run;
        run += c;
    }
}

__global__ void __launch_bounds__(256) key_scatter_kernel(int64_t rows, const uint32_t* keys, uint32_t* offs,
                                                          int32_t* order) {
    for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < rows;
         row += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t pos = atomicAdd(&offs[keys[row]], 1u);
        order[pos] = (int32_t)row;
    }
}

// ------------------------------------------------------------ spectral kernels
struct FftParams {
    FftGeo fft;
    const double2* dtw;  // DCT twiddles exp(-i pi k / 2N)
    int32_t inverse, pad;
    const double* x;
    const double* re;
    const double* im;
    double* xo;
    double* reo;
    double* imo;
    int64_t n;
    int32_t L, lcap;
    const double2* tw;
    double* gbuf;  // non-null: per-CTA row buffers (2 * lcap doubles) in global memory
};

// row buffers of the one-warp transform kernels: shared memory, or this
// CTA's slot of a global scratch for series too long for it
template <bool GMEM>
__device__ __forceinline__ double* row_bufs(unsigned char* smem, double* gbuf, int lcap) {
    return GMEM ? gbuf + (int64_t)blockIdx.x * 2 * (int64_t)lcap : reinterpret_cast<double*>(smem);
}

// Row input of the one-warp transform kernels.  In shared-memory mode with
// 16-byte rows, the next row is prefetched by a TMA bulk copy into the buffer
// the current transform leaves free, so the load overlaps this row's output
// stores (the kernels were bound on these loads at ~6 warps per SM).
struct RowPrefetch {
    uint64_t* bar;
    uint32_t phase, bytes;
    bool bulk;
    __device__ __forceinline__ void start(double* dst, const double* src, int lane) {
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(bar, bytes);
            bulk_g2s(dst, src, bytes, bar);
        }
    }
    __device__ __forceinline__ void wait() {
        mbar_wait(bar, phase);
        phase ^= 1u;
    }
};

template <bool GMEM>
__device__ __forceinline__ RowPrefetch row_prefetch_init(unsigned char* smem, const FftParams& p, double* A, int lane) {
    RowPrefetch rp;
    rp.bar = reinterpret_cast<uint64_t*>(smem + 16 * (size_t)p.lcap);  // after the two buffers
    rp.phase = 0;
    rp.bytes = 8u * (uint32_t)p.L;
    rp.bulk = !GMEM && (p.L % 2 == 0) && ((reinterpret_cast<uintptr_t>(p.x) & 15) == 0);
    if (rp.bulk) {
        if (lane == 0) mbar_init(rp.bar, 1);
        __syncwarp();
        if (blockIdx.x < p.n) rp.start(A, p.x + (int64_t)blockIdx.x * p.L, lane);
    }
    return rp;
}

template <bool GMEM>
__global__ void __launch_bounds__(32) rfft_kernel(const __grid_constant__ FftParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x;
    double* A = row_bufs<GMEM>(smem, p.gbuf, p.lcap);
    double* B = A + p.lcap;
    const int bins = p.L / 2 + 1;
    RowPrefetch rp = row_prefetch_init<GMEM>(smem, p, A, lane);
    for (int64_t row = blockIdx.x; row < p.n; row += gridDim.x) {
        if (rp.bulk) {
            rp.wait();
        } else {
            const double* src = p.x + row * p.L;
            for (int t = lane; t < p.L; t += 32) A[t] = src[t];
        }
        __syncwarp();
        double2* X = rfft_any<true, true>(A, B, p.L, p.fft, p.tw, lane);
        double* freeb = (reinterpret_cast<double*>(X) == A) ? B : A;
        const int64_t next = row + gridDim.x;
        if (rp.bulk && next < p.n) rp.start(freeb, p.x + next * p.L, lane);
        for (int k = lane; k < bins; k += 32) {
            p.reo[row * bins + k] = X[k].x;
            p.imo[row * bins + k] = X[k].y;
        }
        __syncwarp();
        if (rp.bulk) {
            B = reinterpret_cast<double*>(X);
            A = freeb;
        }
    }
}

template <bool GMEM>
__global__ void __launch_bounds__(32) irfft_kernel(const __grid_constant__ FftParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x;
    double2* X = reinterpret_cast<double2*>(row_bufs<GMEM>(smem, p.gbuf, p.lcap));
    double2* O = X + p.lcap / 2;
    const int bins = p.L / 2 + 1;
    // shared-memory rows: the next row's re / im land in the free buffer by
    // cp.async while this row's series is stored
    auto fetch = [&](double2* dst, int64_t row) {
        const double* re = p.re + row * bins;
        const double* im = p.im + row * bins;
        for (int k = lane; k < bins; k += 32) {
            cp_async8(&dst[k].x, re + k);
            cp_async8(&dst[k].y, im + k);
        }
        cp_async_commit();
    };
    if (!GMEM && blockIdx.x < p.n) fetch(X, blockIdx.x);
    for (int64_t row = blockIdx.x; row < p.n; row += gridDim.x) {
        if (GMEM) {
            for (int k = lane; k < bins; k += 32) X[k] = make_double2(p.re[row * bins + k], p.im[row * bins + k]);
        } else {
            cp_async_wait_all();
        }
        __syncwarp();
        double* y = irfft_any<true, true>(X, O, p.L, p.fft, p.tw, lane);
        double2* freeb = (y == reinterpret_cast<double*>(X)) ? O : X;
        const int64_t next = row + gridDim.x;
        if (!GMEM && next < p.n) fetch(freeb, next);
        for (int t = lane; t < p.L; t += 32) p.xo[row * p.L + t] = y[t];
        __syncwarp();
        if (!GMEM) {
            O = reinterpret_cast<double2*>(y);
            X = freeb;
        }
    }
}

// dct_forward / dct_inverse (reference freqtransform.py:91-98), one warp per row
template <bool GMEM>
__global__ void __launch_bounds__(32) dct_kernel(const __grid_constant__ FftParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x;
    double* A = row_bufs<GMEM>(smem, p.gbuf, p.lcap);
    double* B = A + p.lcap;
    RowPrefetch rp = row_prefetch_init<GMEM>(smem, p, A, lane);
    for (int64_t row = blockIdx.x; row < p.n; row += gridDim.x) {
        if (rp.bulk) {
            rp.wait();
        } else {
            const double* src = p.x + row * p.L;
            for (int t = lane; t < p.L; t += 32) A[t] = src[t];
        }
        __syncwarp();
        double* y = p.inverse ? dct3_any(A, B, p.L, p.fft, p.tw, p.dtw, lane)
                              : dct2_any(A, B, p.L, p.fft, p.tw, p.dtw, lane);
        double* freeb = (y == A) ? B : A;
        const int64_t next = row + gridDim.x;
        if (rp.bulk && next < p.n) rp.start(freeb, p.x + next * p.L, lane);
        for (int t = lane; t < p.L; t += 32) p.xo[row * p.L + t] = y[t];
        __syncwarp();
        if (rp.bulk) {
            B = y;
            A = freeb;
        }
    }
}

// CTA-cooperative transforms (sa_fft_cta.cuh): power-of-two complex length
// N = 256 .. 2048, T = N / 8 threads per row.  Shared memory: the FFT's
// exchange buffer (N complex) and a next-row buffer (N + 1 complex) that
// cp.async fills with row r + gridDim while row r is transformed.
struct CtaSmem {
    double2* buf;
    double2* nb;
};
__device__ __forceinline__ CtaSmem cta_smem(unsigned char* smem, int N) {
    double2* b = reinterpret_cast<double2*>(smem);
    return {b, b + N};
}

#ifndef SA_CTA_MINB
#define SA_CTA_MINB 512  // min CTAs per SM x T: a register cap of 65536 / SA_CTA_MINB
#endif

// rfft (freqtransform.py:101-108): real row (N complex) -> bins 0..N
template <int LGN>
__global__ void __launch_bounds__(CtaPlan<LGN>::T, SA_CTA_MINB / CtaPlan<LGN>::T) rfft_cta_kernel(const __grid_constant__ FftParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int T = CtaPlan<LGN>::T;
    const int t = threadIdx.x;
    const int M = p.L >> 1, bins = M + 1;
    const CtaSmem sm = cta_smem(smem, M);
    double2 w[8];
    cta_twiddles<LGN>(w, t, p.tw, LGN + 1);
    auto fetch = [&](int64_t row) {
        const double2* xr = reinterpret_cast<const double2*>(p.x + row * p.L);
        for (int i = t; i < M; i += T) cp_async16(&sm.nb[i], xr + i);
        cp_async_commit();
    };
    double2 ws[8];  // split twiddles W_L^k, k = t + m T
#pragma unroll
    for (int m = 0; m < 8; ++m) ws[m] = __ldg(&p.tw[t + m * T]);
    if (blockIdx.x < p.n) fetch(blockIdx.x);
    for (int64_t row = blockIdx.x; row < p.n; row += gridDim.x) {
        double2 v[8];
        cp_async_wait_all();
        __syncthreads();
#pragma unroll
        for (int m = 0; m < 8; ++m) v[m] = sm.nb[t + m * T];
        __syncthreads();
        if (row + gridDim.x < p.n) fetch(row + gridDim.x);
        cta_fft<LGN>(v, sm.buf, t, w);
        __syncthreads();
#pragma unroll
        for (int m = 0; m < 8; ++m) sm.buf[t + m * T] = v[m];
        __syncthreads();
        double* re = p.reo + row * bins;
        double* im = p.imo + row * bins;
#pragma unroll 4
        for (int m = 0; m < 8; ++m) {
            const int k = t + m * T;
            double2 X = cta_split(sm.buf[k], sm.buf[k == 0 ? 0 : M - k], ws[m]);
            if (k == 0) X.y = 0.0;
            __stcs(re + k, X.x);
            __stcs(im + k, X.y);
        }
        if (t == 0) {
            const double2 X = cta_split(sm.buf[0], sm.buf[0], __ldg(&p.tw[M]));
            __stcs(re + M, X.x);
            __stcs(im + M, 0.0);
        }
    }
}

// irfft (freqtransform.py:110-116): bins 0..N (separate re / im rows) -> real row
template <int LGN>
__global__ void __launch_bounds__(CtaPlan<LGN>::T, SA_CTA_MINB / CtaPlan<LGN>::T) irfft_cta_kernel(const __grid_constant__ FftParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int T = CtaPlan<LGN>::T;
    const int t = threadIdx.x;
    const int M = p.L >> 1, bins = M + 1;
    const CtaSmem sm = cta_smem(smem, M);
    double2 w[8];
    cta_twiddles<LGN>(w, t, p.tw, LGN + 1);
    const double s = 1.0 / (double)M;
    auto fetch = [&](int64_t row) {  // interleave re / im into complex bins
        const double* re = p.re + row * bins;
        const double* im = p.im + row * bins;
        for (int k = t; k < bins; k += T) {
            cp_async8(&sm.nb[k].x, re + k);
            cp_async8(&sm.nb[k].y, im + k);
        }
        cp_async_commit();
    };
    double2 ws[8];  // fold twiddles W_L^k, k = t + m T
#pragma unroll
    for (int m = 0; m < 8; ++m) ws[m] = __ldg(&p.tw[t + m * T]);
    if (blockIdx.x < p.n) fetch(blockIdx.x);
    for (int64_t row = blockIdx.x; row < p.n; row += gridDim.x) {
        double2 v[8];
        cp_async_wait_all();
        __syncthreads();
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const int k = t + m * T;
            v[m] = cta_fold(sm.nb[k], sm.nb[M - k], ws[m], k == 0);
        }
        __syncthreads();
        if (row + gridDim.x < p.n) fetch(row + gridDim.x);
        cta_fft<LGN>(v, sm.buf, t, w);
        double2* xo = reinterpret_cast<double2*>(p.xo + row * p.L);
#pragma unroll
        for (int m = 0; m < 8; ++m) __stcs(xo + t + m * T, make_double2(v[m].x * s, -(v[m].y * s)));
    }
}

// DCT-II / DCT-III (orthonormal, freqtransform.py:91-98) of length Lr = 2N,
// dct2_any / dct3_any's formulas; the Makhoul permutation is applied by the
// row fetch (II: v[i] = x[2i], v[Lr-1-i] = x[2i+1]) or the row store (III).
template <int LGN>
__global__ void __launch_bounds__(CtaPlan<LGN>::T, SA_CTA_MINB / CtaPlan<LGN>::T) dct2_cta_kernel(const __grid_constant__ FftParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int T = CtaPlan<LGN>::T;
    const int t = threadIdx.x;
    const int Lr = p.L, N = Lr >> 1;
    const CtaSmem sm = cta_smem(smem, N);
    double* nbd = reinterpret_cast<double*>(sm.nb);
    double2 w[8];
    cta_twiddles<LGN>(w, t, p.tw, LGN + 1);
    auto fetch = [&](int64_t row) {
        const double* xr = p.x + row * Lr;
        for (int i = t; i < N; i += T) {
            cp_async8(&nbd[i], xr + 2 * i);
            cp_async8(&nbd[Lr - 1 - i], xr + 2 * i + 1);
        }
        cp_async_commit();
    };
    if (blockIdx.x < p.n) fetch(blockIdx.x);
    const double g0 = 1.0 / sqrt((double)Lr), gk = sqrt(2.0 / (double)Lr);
    for (int64_t row = blockIdx.x; row < p.n; row += gridDim.x) {
        double2 v[8];
        cp_async_wait_all();
        __syncthreads();
#pragma unroll
        for (int m = 0; m < 8; ++m) v[m] = sm.nb[t + m * T];
        __syncthreads();
        if (row + gridDim.x < p.n) fetch(row + gridDim.x);
        cta_fft<LGN>(v, sm.buf, t, w);
        __syncthreads();
#pragma unroll
        for (int m = 0; m < 8; ++m) sm.buf[t + m * T] = v[m];
        __syncthreads();
        double* y = p.xo + row * Lr;
#pragma unroll 2
        for (int m = 0; m < 8; ++m) {
            const int k = t + m * T;
            double2 X = cta_split(sm.buf[k], sm.buf[k == 0 ? 0 : N - k], __ldg(&p.tw[k]));
            if (k == 0) X.y = 0.0;
            const double2 w = __ldg(&p.dtw[k]);
            __stcs(y + k, (k == 0 ? g0 : gk) * (X.x * w.x - X.y * w.y));
            if (k > 0) {
                const double2 w2 = __ldg(&p.dtw[Lr - k]);  // V[Lr-k] = conj(V[k])
                __stcs(y + Lr - k, gk * (X.x * w2.x + X.y * w2.y));
            }
        }
        if (t == 0) {
            double2 X = cta_split(sm.buf[0], sm.buf[0], __ldg(&p.tw[N]));
            X.y = 0.0;
            const double2 w = __ldg(&p.dtw[N]);
            __stcs(y + N, gk * (X.x * w.x - X.y * w.y));
        }
    }
}

template <int LGN>
__global__ void __launch_bounds__(CtaPlan<LGN>::T, SA_CTA_MINB / CtaPlan<LGN>::T) dct3_cta_kernel(const __grid_constant__ FftParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int T = CtaPlan<LGN>::T;
    const int t = threadIdx.x;
    const int Lr = p.L, N = Lr >> 1;
    const CtaSmem sm = cta_smem(smem, N);
    const double* nbd = reinterpret_cast<const double*>(sm.nb);
    const double* xb = reinterpret_cast<const double*>(sm.buf);
    double2 w[8];
    cta_twiddles<LGN>(w, t, p.tw, LGN + 1);
    auto fetch = [&](int64_t row) {
        const double2* yr = reinterpret_cast<const double2*>(p.x + row * Lr);
        for (int i = t; i < N; i += T) cp_async16(&sm.nb[i], yr + i);
        cp_async_commit();
    };
    if (blockIdx.x < p.n) fetch(blockIdx.x);
    const double i0 = sqrt((double)Lr), ik = sqrt((double)Lr / 2.0);
    const double s = 1.0 / (double)N;
    auto V = [&](int q) {  // V[q] = e^{+i pi q / 2Lr} (S[q] - i S[Lr-q]), q <= N
        const double sk = nbd[q] * (q == 0 ? i0 : ik);
        const double snk = (q == 0) ? 0.0 : nbd[Lr - q] * ik;
        double2 w = __ldg(&p.dtw[q]);
        w.y = -w.y;
        return cmul(make_double2(sk, -snk), w);
    };
    for (int64_t row = blockIdx.x; row < p.n; row += gridDim.x) {
        double2 v[8];
        cp_async_wait_all();
        __syncthreads();
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const int k = t + m * T;
            v[m] = cta_fold(V(k), V(N - k), __ldg(&p.tw[k]), k == 0);
        }
        __syncthreads();
        if (row + gridDim.x < p.n) fetch(row + gridDim.x);
        cta_fft<LGN>(v, sm.buf, t, w);
        __syncthreads();
#pragma unroll
        for (int m = 0; m < 8; ++m) sm.buf[t + m * T] = make_double2(v[m].x * s, -(v[m].y * s));
        __syncthreads();
        double2* xo = reinterpret_cast<double2*>(p.xo + row * Lr);
        for (int i = t; i < N; i += T) __stcs(xo + i, make_double2(xb[i], xb[Lr - 1 - i]));
    }
}

// Spectral-only chains (every stage FrequencyMask / RandomSinusoid, e.g.
// BASELINE config 3) on the CTA FFT: one CTA per row, rfft -> the fired
// stages' perturbations on the bins -> irfft, the row never leaving the SM
// (freqaugment.py:37-47, 131-170 + BASELINE M6; the warp chain's op_spectral
// with spectrum residency).  Warp 0 draws each stage's gate and scalars (one
// lane per stage, SStream); rows none of whose stages fire are copied.
// Gates and scalar draws of a spectral-only chain, one thread per (row,
// stage): the stage's stream (core.py:77-82), its gate (core.py:235), the
// mask start (freqaugment.py:162-170) or the sinusoid bin / phase increment
// (BASELINE M6).  A parallel pre-pass, so the CTA kernel's rows never wait
// on a serial draw section; each row's entries are cp.async-prefetched with
// the row itself.
struct SpecDraw {
    double2 add;  // sinusoid increment
    int32_t pos;  // mask start / sinusoid bin
    int32_t fire;
    int64_t pad;
};
__global__ void __launch_bounds__(256) spectral_draw_kernel(const __grid_constant__ ChainParams p,
                                                            SpecDraw* __restrict__ out) {
    const int L = (int)p.len_in, bins = L / 2 + 1;
    const int64_t total = p.rows_out * (int64_t)p.ns;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / p.ns;
        const int j = (int)(i - row * p.ns);
        const DevStage& st = p.st[j];
        uint64_t k0, k1;
        derive_key(p.seed, (uint64_t)st.index, (uint64_t)(p.offset + row), k0, k1);
        SStream s;
        s_init(s, k0, k1);
        SpecDraw d;
        d.add = make_double2(0.0, 0.0);
        d.pos = 0;
        d.pad = 0;
        const bool f = s_next_double(s) < st.prob && !spectral_noop(st);
        d.fire = f ? 1 : 0;
        if (f && st.op == SA_OP_FREQ_MASK) {
            const int wd = (int)st.i[0];
            int start = (int)s_bounded(s, (uint32_t)(bins - 1)) - wd / 2;
            if (start < 0) start = 0;
            if (start > bins - wd) start = bins - wd;
            d.pos = start;
        } else if (f) {  // SA_OP_SINUSOID
            const int mb = (int)st.i[0];
            const int b = mb + (int)s_bounded(s, (uint32_t)(bins - mb - 1));
            const double phi = (2.0 * 3.14159265358979323846) * s_next_double(s);
            const double A = st.f[0];
            d.pos = b;
            if (b == 0 || b == bins - 1) {
                d.add = make_double2((A * (double)L) * cos(phi), 0.0);
            } else {
                const double h = (A * (double)L) * 0.5;
                d.add = make_double2(h * cos(phi), h * sin(phi));
            }
        }
        out[i] = d;
    }
}

#ifndef SA_SPEC_THREADS
#define SA_SPEC_THREADS 640  // resident threads per SM the register budget targets
#endif
template <int LGN>
__global__ void __launch_bounds__(CtaPlan<LGN>::T, SA_SPEC_THREADS / CtaPlan<LGN>::T) spectral_cta_kernel(const __grid_constant__ ChainParams p,
                                                           const double2* __restrict__ tw,
                                                           const SpecDraw* __restrict__ draws) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int T = CtaPlan<LGN>::T, N = 1 << LGN;
    const int t = threadIdx.x;
    const int L = 2 * N, bins = N + 1;
    const CtaSmem sm = cta_smem(smem, N);
    __shared__ __align__(16) SpecDraw s_tab[2][64];  // this / next row's draws, stage j
    double2 w[8];
    cta_twiddles<LGN>(w, t, tw, LGN + 1);
    const double2 wn = __ldg(&tw[N]);
    auto fetch = [&](int64_t row, int b) {
        const double2* xr = reinterpret_cast<const double2*>(p.in + row * L);
        for (int i = t; i < N; i += T) cp_async16(&sm.nb[i], xr + i);
        const char* dr = reinterpret_cast<const char*>(draws + row * p.ns);
        char* ds = reinterpret_cast<char*>(&s_tab[b][0]);
        for (int i = t; i < 2 * p.ns; i += T) cp_async16(ds + 16 * i, dr + 16 * i);
        cp_async_commit();
    };
    if (blockIdx.x < p.rows_out) fetch(blockIdx.x, 0);
    bool bad = false;
    int cb = 0;  // s_tab buffer of the current row
    for (int64_t row = blockIdx.x; row < p.rows_out; row += gridDim.x, cb ^= 1) {
        cp_async_wait_all();
        __syncthreads();
        double2 v[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            v[m] = sm.nb[t + m * T];
            bad |= nonfinite(v[m].x) | nonfinite(v[m].y);  // Batch invariant (core.py:104)
        }
        uint64_t fire = 0;
        for (int j = 0; j < p.ns; ++j) fire |= (uint64_t)(s_tab[cb][j].fire != 0) << j;
        __syncthreads();
        if (row + gridDim.x < p.rows_out) fetch(row + gridDim.x, cb ^ 1);
        double2* xo = reinterpret_cast<double2*>(p.out + row * L);
        if (!fire) {
#pragma unroll
            for (int m = 0; m < 8; ++m) __stcs(xo + t + m * T, v[m]);
            continue;
        }
        cta_fft<LGN>(v, sm.buf, t, w);
        __syncthreads();
#pragma unroll
        for (int m = 0; m < 8; ++m) sm.buf[t + m * T] = v[m];
        __syncthreads();
        // Bin pairs (k, N - k) that no fired stage touches go straight to the
        // inverse FFT's input: fold(split(Z)) = conj(Z) there (irfft(rfft(x))
        // = x), so only the pairs a mask / sinusoid reaches run the split, the
        // stages and the fold -- on both bins of the pair, in this thread (the
        // Nyquist bin N pairs with k = 0).  Same formulas and pins as
        // rfft_any / _apply / irfft_any; untouched bins skip rounding-level work.
        // bit m: pair of bin t + m T touched by a fired stage.  Bins [pos, end)
        // hold k = t + m T for m in [ceil((pos - t) / T), ceil((end - t) / T))
        // and kc = N - k for m in [ceil((N + 1 - end - t) / T), ceil((N + 1 - pos - t) / T))
        // (floor division by the power of two T: arithmetic shift)
        constexpr int LGT = LGN - 3;
        auto mbits = [&](int lo, int hi) -> uint32_t {  // m in [ceil(lo / T), ceil(hi / T)) within 0..7
            int a = (lo + T - 1) >> LGT, b = (hi + T - 1) >> LGT;
            a = a < 0 ? 0 : (a > 8 ? 8 : a);
            b = b < 0 ? 0 : (b > 8 ? 8 : b);
            return ((1u << b) - 1u) & ~((1u << a) - 1u);
        };
        uint32_t affm = 0;
        for (uint64_t f = fire; f; f &= f - 1) {
            const int j = __ffsll((long long)f) - 1;
            const int pos = s_tab[cb][j].pos;
            const int end = p.st[j].op == SA_OP_FREQ_MASK ? pos + (int)p.st[j].i[0] : pos + 1;
            affm |= mbits(pos - t, end - t) | mbits(N + 1 - end - t, N + 1 - pos - t);
        }
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const int k = t + m * T, kc = N - k;
            if (((affm >> m) & 1u) == 0u) {
                v[m] = make_double2(v[m].x, -v[m].y);
            } else {
                const double2 wk = __ldg(&tw[k]);  // only touched pairs: L1, not registers (5 CTAs / SM)
                const double2 zk = v[m], zc = sm.buf[k == 0 ? 0 : kc];
                double2 a = cta_split(zk, zc, wk);
                double2 c = cta_split(zc, zk, k == 0 ? wn : make_double2(-wk.x, wk.y));  // W_L^{N-k} = -conj(W_L^k)
                if (k == 0) {  // DC / Nyquist imaginary parts pinned (freqaugment.py:40-45)
                    a.y = 0.0;
                    c.y = 0.0;
                }
                for (uint64_t f = fire; f; f &= f - 1) {  // stages in chain order
                    const int j = __ffsll((long long)f) - 1;
                    const int pos = s_tab[cb][j].pos;
                    if (p.st[j].op == SA_OP_FREQ_MASK) {
                        const int end = pos + (int)p.st[j].i[0];
                        if (k >= pos && k < end) a = make_double2(0.0, 0.0);
                        if (kc >= pos && kc < end) c = make_double2(0.0, 0.0);
                    } else {
                        const double2 ad = s_tab[cb][j].add;
                        if (k == pos) {
                            a.x = a.x + ad.x;
                            if (pos != 0) a.y = a.y + ad.y;
                        }
                        if (kc == pos) {
                            c.x = c.x + ad.x;
                            if (pos != N) c.y = c.y + ad.y;
                        }
                    }
                }
                v[m] = cta_fold(a, c, wk, k == 0);
            }
        }
        cta_fft<LGN>(v, sm.buf, t, w);
        const double sc = 1.0 / (double)N;
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const double2 o = make_double2(v[m].x * sc, -(v[m].y * sc));
            bad |= nonfinite(o.x) | nonfinite(o.y);
            __stcs(xo + t + m * T, o);
        }
    }
    if (__any_sync(SA_FULL, bad) && (t & 31) == 0) atomicOr(p.flags, SA_FLAG_NONFINITE);
}

// Gather-only chains (every stage SpeedWarp / Resize / Convolve / Rotate /
// Reverse, e.g. BASELINE config 4) on a CTA per row.  The warp-per-row chain
// kernel holds two row buffers per warp, so at L = 1,500 only 8 rows (8
// warps) fit an SM and the gathers' dependent FP64 chains are latency bound.
// Here the gates and SpeedWarp's speed draws come from a parallel pre-pass
// (gather_draw_kernel: one thread per (row, stage), the stage's numpy stream
// restated by SStream) and GT threads share each row: the same two buffers
// per row, GT / 32 times the warps, and no RNG or lockstep code in the main
// kernel (few registers).  Every operator's arithmetic is the chain kernel's
// (same formulas, same order), so results are bitwise the same.
constexpr int kGatherMaxSpeeds = 8;  // SpeedWarp n_speed_change <= 7
#ifndef SA_GATHER_THREADS
#define SA_GATHER_THREADS 128
#endif
constexpr int kGatherThreads = SA_GATHER_THREADS;  // threads per row
struct GatherDraw {
    double v[kGatherMaxSpeeds];  // SpeedWarp: speeds 1 + (R - 1) random()
    int32_t fire;
    int32_t pad[3];
};
__global__ void __launch_bounds__(256) gather_draw_kernel(const __grid_constant__ ChainParams p,
                                                          GatherDraw* __restrict__ out) {
    const int64_t total = p.rows_out * (int64_t)p.ns;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / p.ns;
        const int j = (int)(i - row * p.ns);
        const DevStage& st = p.st[j];
        uint64_t k0, k1;
        derive_key(p.seed, (uint64_t)st.index, (uint64_t)(p.offset + row), k0, k1);
        SStream s;
        s_init(s, k0, k1);
        GatherDraw d;
        d.fire = s_next_double(s) < st.prob ? 1 : 0;  // core.py:235
        if (d.fire && st.op == SA_OP_SPEED_WARP) {
            const int K = (int)st.i[0];
            const double lo = 1.0, range = st.f[0] - lo;
            for (int m = 0; m <= K && m < kGatherMaxSpeeds; ++m) d.v[m] = lo + range * s_next_double(s);
        }
        out[i] = d;
    }
}

template <int GT>
__global__ void __launch_bounds__(GT) gather_cta_kernel(const __grid_constant__ ChainParams p,
                                                        const GatherDraw* __restrict__ draws) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x;
    double* bufs = reinterpret_cast<double*>(smem);
    double* sw_base = bufs + 2 * (size_t)p.lcap;  // SpeedWarp cumulative bases, then f
    int32_t* sw_sb = reinterpret_cast<int32_t*>(sw_base + kGatherMaxSpeeds + 2);  // segment starts
    GatherDraw* s_dr = reinterpret_cast<GatherDraw*>(sw_sb + kGatherMaxSpeeds + 8);  // this row's draws (16-B aligned)
    Finite bad, bad2;  // two independent accumulation chains
    double* cur = bufs;
    double* oth = bufs + p.lcap;
    // rows (and their draws) arrive by cp.async: the next row is fetched into
    // the free buffer while the current one is stored
    const bool vec = ((p.len_in & 1) | (reinterpret_cast<uintptr_t>(p.in) & 15u)) == 0;
    auto fetch = [&](int64_t r, double* dst) {
        const double* src = p.in + r * (int64_t)p.len_in;
        if (vec) {
            for (int t = tid; t < p.len_in / 2; t += GT) cp_async16(dst + 2 * t, src + 2 * t);
        } else {
            for (int t = tid; t < p.len_in; t += GT) cp_async8(dst + t, src + t);
        }
        const char* g = reinterpret_cast<const char*>(draws + r * p.ns);
        for (int i = tid; i < p.ns * (int)(sizeof(GatherDraw) / 16); i += GT)
            cp_async16(reinterpret_cast<char*>(s_dr) + 16 * i, g + 16 * i);
        cp_async_commit();
    };
    if (blockIdx.x < p.rows_out) fetch(blockIdx.x, cur);
    for (int64_t row = blockIdx.x; row < p.rows_out; row += gridDim.x) {
        cp_async_wait_all();
        __syncthreads();
        int L = p.len_in;
        for (int t = tid; t < L / 2; t += GT) {  // Batch invariant (core.py:104)
            const double2 v = reinterpret_cast<const double2*>(cur)[t];
            bad.chk(v.x);
            bad2.chk(v.y);
        }
        if (L & 1) {
            if (tid == 0) bad.chk(cur[L - 1]);
        }
        const GatherDraw* dr = s_dr;
        for (int j = 0; j < p.ns; ++j) {
            const DevStage& st = p.st[j];
            if (!dr[j].fire) continue;  // uniform across the CTA
            switch (st.op) {
                case SA_OP_ROTATE:  // basic.py:70-71
                    for (int t = tid; t < L; t += GT) cur[t] = -cur[t];
                    __syncthreads();
                    break;
                case SA_OP_REVERSE:  // basic.py:113-114
                    for (int t = tid; t < L; t += GT) oth[t] = cur[L - 1 - t];
                    __syncthreads();
                    swapbuf(cur, oth);
                    break;
                case SA_OP_RESIZE: {  // basic.py Resize: np.interp on linspace(0, L - 1, T)
                    const int T = (int)st.i[0];
                    if (T == L) break;
                    const Linspace ls(0.0, (double)L - 1.0, T);
                    for (int t = tid; t < T; t += GT) {
                        const double v = ls.fast() ? interp_grid_fast(ls.at_fast(t), cur, L) : interp_grid(ls.at(t), cur, L);
                        oth[t] = v;
                        bad.chk(v);
                    }
                    __syncthreads();
                    swapbuf(cur, oth);
                    L = T;
                    break;
                }
                case SA_OP_CONVOLVE: {  // BASELINE M4: y_t = sum_k taps[k] x[clip(t + k - S/2)], k in order
                    const double* taps = p.aux + st.aux_off;
                    const int S = st.aux_len, h = S / 2;
                    if (S == 7 && L >= 16) {
                        // lane pairs as convolve7: outputs t, t + 1 (t even) from five
                        // aligned 16-byte loads of x[t - 4 .. t + 5]; edges clamped
                        double c[7];
#pragma unroll
                        for (int k = 0; k < 7; ++k) c[k] = taps[k];
                        const int tmax = L - 6;  // last interior pair start
                        const double2* c2 = reinterpret_cast<const double2*>(cur);
                        for (int t = 4 + 2 * tid; t <= tmax; t += 2 * GT) {
                            double2 v[5];
#pragma unroll
                            for (int m = 0; m < 5; ++m) v[m] = c2[(t - 4) / 2 + m];
                            const double x[10] = {v[0].x, v[0].y, v[1].x, v[1].y, v[2].x,
                                                  v[2].y, v[3].x, v[3].y, v[4].x, v[4].y};
                            double a0 = 0.0, a1 = 0.0;
#pragma unroll
                            for (int k = 0; k < 7; ++k) {
                                a0 = a0 + c[k] * x[1 + k];
                                a1 = a1 + c[k] * x[2 + k];
                            }
                            reinterpret_cast<double2*>(oth)[t / 2] = make_double2(a0, a1);
                            bad.chk(a0);
                            bad2.chk(a1);
                        }
                        const int e0 = 4 + 2 * ((tmax - 4) / 2) + 2;
                        for (int i = tid; i < 4 + (L - e0); i += GT) {
                            const int t = i < 4 ? i : e0 + (i - 4);
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
                        __syncthreads();
                        swapbuf(cur, oth);
                        break;
                    }
                    for (int t = tid; t < L; t += GT) {
                        double acc = 0.0;
                        if (t >= h && t + S - 1 - h <= L - 1) {
                            const double* pa = cur + t - h;
                            for (int k = 0; k < S; ++k) acc = acc + taps[k] * pa[k];
                        } else {
                            for (int k = 0; k < S; ++k) {
                                int u = t + k - h;
                                u = u < 0 ? 0 : (u > L - 1 ? L - 1 : u);
                                acc = acc + taps[k] * cur[u];
                            }
                        }
                        oth[t] = acc;
                        bad.chk(acc);
                    }
                    __syncthreads();
                    swapbuf(cur, oth);
                    break;
                }
                case SA_OP_SPEED_WARP: {  // BASELINE M5 (the chain kernel's op_speed_warp)
                    const int K = (int)st.i[0];
                    if (K == 0 || st.f[0] == 1.0) break;
                    const double* speeds = dr[j].v;
                    for (int m = tid; m <= K + 1; m += GT) sw_sb[m] = m <= K ? seg_start(m, L, K) : L;
                    __syncthreads();
                    if (tid == 0) {
                        double acc = 0.0;
                        sw_base[0] = 0.0;
                        for (int m = 0; m < K; ++m) {
                            acc = acc + speeds[m] * (double)(sw_sb[m + 1] - sw_sb[m]);
                            sw_base[m + 1] = acc;
                        }
                        int mm = 0;
                        while (mm < K && L - 1 >= sw_sb[mm + 1]) ++mm;
                        sw_base[kGatherMaxSpeeds] = ((double)L - 1.0) / (sw_base[mm] + speeds[mm] * (double)(L - 1 - sw_sb[mm]));
                    }
                    __syncthreads();
                    const double f = sw_base[kGatherMaxSpeeds];
                    for (int m = 0; m <= K; ++m) {  // warped positions, segment by segment
                        const int sbm = sw_sb[m], sn = sw_sb[m + 1];
                        const double bm = sw_base[m], spm = speeds[m];
                        for (int t = sbm + tid; t < sn; t += GT)
                            oth[t] = (t == L - 1) ? (double)L - 1.0 : (bm + spm * (double)(t - sbm)) * f;
                    }
                    __syncthreads();
                    const bool cubic = st.i[1] != 0;
                    const double x0 = cur[0], xl = cur[L - 1];
                    for (int t = tid; t < L; t += GT) {
                        const double tau = oth[t];
                        int jj = (int)floor(tau);
                        jj = max(0, min(jj, L - 2));
                        const double fr = tau - (double)jj;
                        const double p1 = cur[jj], p2 = cur[jj + 1];
                        double y;
                        if (cubic) {
                            const double p0 = cur[max(jj - 1, 0)], p3 = cur[min(jj + 2, L - 1)];
                            const double a = ((-0.5 * p0 + 1.5 * p1) - 1.5 * p2) + 0.5 * p3;
                            const double b = ((p0 - 2.5 * p1) + 2.0 * p2) - 0.5 * p3;
                            const double c = -0.5 * p0 + 0.5 * p2;
                            y = ((a * fr + b) * fr + c) * fr + p1;
                        } else {
                            y = p1 + (p2 - p1) * fr;
                        }
                        y = (tau >= (double)(L - 1)) ? xl : y;
                        y = (tau <= 0.0) ? x0 : y;
                        oth[t] = y;  // same thread, same index as its tau
                        bad.chk(y);
                    }
                    __syncthreads();
                    swapbuf(cur, oth);
                    break;
                }
                default: break;
            }
        }
        __syncthreads();  // the draws and the free buffer are no longer read
        if (row + gridDim.x < p.rows_out) fetch(row + gridDim.x, oth);
        double* dst = p.out + row * (int64_t)p.len_out;
        if (((p.len_out & 1) | (reinterpret_cast<uintptr_t>(dst) & 15u) | (reinterpret_cast<uintptr_t>(cur) & 15u)) == 0) {
            for (int t = tid; t < p.len_out / 2; t += GT)
                __stcs(&reinterpret_cast<double2*>(dst)[t], reinterpret_cast<const double2*>(cur)[t]);
        } else {
            for (int t = tid; t < p.len_out; t += GT) __stcs(&dst[t], cur[t]);
        }
        swapbuf(cur, oth);  // the prefetched row (the loop head waits for it and barriers)
    }
    if (__any_sync(SA_FULL, bad.any() || bad2.any()) && (tid & 31) == 0) atomicOr(p.flags, SA_FLAG_NONFINITE);
}

// DTW (reference dtw.py:40-106) -----------------------
struct DtwParams {
    const double* a;
    const double* b;
    double* dist;
    double* acc;      // path mode: n x m workspace
    int32_t* path;    // path mode: 2 * (n + m) ints
    int32_t* path_len;
    int64_t pairs;
    int32_t n, m;
    int32_t stage_b;  // 1: dtw_warp copies b into shared memory
    double* gprow;    // non-null: the previous-row buffer in global memory (len_b too long for smem)
};

// one warp per pair: distance only
template <bool GMEM>
__global__ void __launch_bounds__(32) dtw_batch_kernel(const __grid_constant__ DtwParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* prow = GMEM ? p.gprow + (int64_t)blockIdx.x * p.m : reinterpret_cast<double*>(smem);
    for (int64_t q = blockIdx.x; q < p.pairs; q += gridDim.x) {
        const double d = dtw_warp(p.a + q * p.n, p.n, p.b + q * p.m, p.m, prow, nullptr, threadIdx.x, p.stage_b != 0);
        if (threadIdx.x == 0) p.dist[q] = d;
        __syncwarp();
    }
}

// one pair with the full matrix and the reference's backtracked path
template <bool GMEM>
__global__ void __launch_bounds__(32) dtw_path_kernel(const __grid_constant__ DtwParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* prow = GMEM ? p.gprow : reinterpret_cast<double*>(smem);
    const double d = dtw_warp(p.a, p.n, p.b, p.m, prow, p.acc, threadIdx.x, p.stage_b != 0);
    __syncwarp();
    __threadfence_block();
    if (threadIdx.x == 0) {
        p.dist[0] = d;
        p.path_len[0] = dtw_backtrack(p.acc, p.n, p.m, p.path);
    }
}

// ------------------------------------------------------------ text codec (dataset IO)
__global__ void __launch_bounds__(256) repr_values_kernel(const double* __restrict__ v, int64_t n, char* out,
                                                          int32_t* len) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        char buf[32];
        const int k = repr_format(v[i], buf);
        for (int t = 0; t < k; ++t) out[i * 32 + t] = buf[t];
        len[i] = k;
    }
}

__global__ void __launch_bounds__(256) parse_values_kernel(const char* __restrict__ text, const int64_t* __restrict__ off,
                                                           int64_t n, double* out, int32_t* ok, char* scratch) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double v = 0.0;
        const bool good = parse_field(text, off[i], off[i + 1], scratch, &v);
        out[i] = v;
        ok[i] = good ? 1 : 0;
    }
}

struct SpecParams {
    DevStage st;
    uint64_t seed;
    int64_t offset;
    const double* re;
    const double* im;
    double* reo;
    double* imo;
    int64_t n;
    int32_t L, lcap;
    double* gbuf;  // non-null: per-CTA spectrum + scratch in global memory
};

// SpectralAugmenter.augment_spectrum (freqaugment.py:49-76)
template <bool GMEM>
__global__ void __launch_bounds__(32) spectrum_kernel(const __grid_constant__ SpecParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x;
    double2* X = reinterpret_cast<double2*>(row_bufs<GMEM>(smem, p.gbuf, p.lcap));
    double* scratch = reinterpret_cast<double*>(X + p.lcap / 2);
    uint64_t* win = GMEM ? reinterpret_cast<uint64_t*>(smem) : reinterpret_cast<uint64_t*>(scratch + p.lcap);
    uint64_t* c = win + SA_WIN;
    Warp w;
    w.lane = lane;
    w.zig = g_zig;
    w.win = win;
    const int bins = p.L / 2 + 1;
    for (int64_t row = blockIdx.x; row < p.n; row += gridDim.x) {
        for (int k = lane; k < bins; k += 32) X[k] = make_double2(p.re[row * bins + k], p.im[row * bins + k]);
        uint64_t k0, k1, o0, o1, o2, o3;
        derive_key(p.seed, (uint64_t)p.st.index, (uint64_t)(p.offset + row), k0, k1);
        philox(k0, k1, 1, o0, o1, o2, o3);
        if (lane == 0) { c[0] = o0; c[1] = o1; c[2] = o2; c[3] = o3; }
        __syncwarp();
        if (u53(o0) < p.st.prob && !spectral_noop(p.st)) {
            WStream s;
            s.k0 = k0; s.k1 = k1; s.win = c; s.winbuf = win; s.wb = 0; s.wn = 4; s.wpos = 1;
            s.has32 = 0; s.u32 = 0;
            perturb_spectrum(p.st, s, X, p.L, scratch, w);
        }
        for (int k = lane; k < bins; k += 32) {
            p.reo[row * bins + k] = X[k].x;
            p.imo[row * bins + k] = X[k].y;
        }
        __syncwarp();
    }
}

}  // namespace sa

// ====================================================================== host
using namespace sa;

namespace {

thread_local std::string g_err;
int64_t g_launches = 0;
std::mutex g_mu;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char* what) {
    return fail(SA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define SA_CUDA(call)                                 \
    do {                                              \
        cudaError_t e_ = (call);                      \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

struct DeviceState {
    bool ready = false;
    int sms = 0;
    size_t smem_optin = 0;
    std::map<int, double2*> twiddles;  // by length
    // host-buffer path (sa_host_stage.inc): slot streams and flag words
    static constexpr int NS = 3;  // pipeline depth (copy-in / H2D+kernel+D2H / copy-out in flight)
    cudaStream_t hs[NS] = {nullptr, nullptr, nullptr};
    uint32_t* dflags = nullptr;
};
// Per-device state in a fixed array: lookups never reallocate, so readers
// need no lock; initialisation and the caches inside are guarded by g_mu,
// the host-buffer pipeline (streams + staging buffers) by its own mutex.
constexpr int kMaxDevices = 64;
DeviceState g_dev_state[kMaxDevices];
std::mutex g_host_mu[kMaxDevices];

DeviceState& dev_state(int dev) { return g_dev_state[dev < 0 ? 0 : (dev >= kMaxDevices ? kMaxDevices - 1 : dev)]; }

// Stream-ordered scratch (scheduling buffers, global row buffers, dataset
// intermediates) comes from a private memory pool per device, so the host
// application's default pool keeps its own release policy.  Up to 1 GiB stays
// mapped between calls (the default threshold of 0 unmaps at every
// synchronisation and the next allocation pays a remap: 20-60 ms host stalls
// were measured); larger transient buffers are returned at synchronisation.
cudaMemPool_t g_pool[kMaxDevices];
std::once_flag g_pool_once[kMaxDevices];
cudaError_t g_pool_err[kMaxDevices];

cudaError_t sa_malloc_async(void** p, size_t bytes, cudaStream_t st) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const int d = dev < 0 ? 0 : (dev >= kMaxDevices ? kMaxDevices - 1 : dev);
    std::call_once(g_pool_once[d], [&] {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        g_pool_err[d] = cudaMemPoolCreate(&g_pool[d], &props);
        if (g_pool_err[d] == cudaSuccess) {
            uint64_t keep = 1ull << 30;
            g_pool_err[d] = cudaMemPoolSetAttribute(g_pool[d], cudaMemPoolAttrReleaseThreshold, &keep);
        }
    });
    if (g_pool_err[d] != cudaSuccess) return g_pool_err[d];
    return cudaMallocFromPoolAsync(p, bytes, g_pool[d], st);
}

int current_device_id() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

int current_device(int* dev) {
    SA_CUDA(cudaGetDevice(dev));
    return SA_OK;
}

int init_device(int dev) {
    std::lock_guard<std::mutex> lk(g_mu);
    DeviceState& ds = dev_state(dev);
    if (ds.ready) return SA_OK;
    int prev;
    SA_CUDA(cudaGetDevice(&prev));
    SA_CUDA(cudaSetDevice(dev));
    static const uint64_t ki[256] = SA_ZIG_KI_DOUBLE_INIT;
    static const uint64_t wi[256] = SA_ZIG_WI_DOUBLE_INIT;
    static const uint64_t fi[256] = SA_ZIG_FI_DOUBLE_INIT;
    ZigEntry zig[256];
    double fid[256];
    for (int k = 0; k < 256; ++k) {
        zig[k].ki = ki[k];
        std::memcpy(&zig[k].wi, &wi[k], 8);
        std::memcpy(&fid[k], &fi[k], 8);
    }
    SA_CUDA(cudaMemcpyToSymbol(g_zig, zig, sizeof(zig)));
    SA_CUDA(cudaMemcpyToSymbol(g_fi, fid, sizeof(fid)));
    SA_CUDA(cudaDeviceGetAttribute(&ds.sms, cudaDevAttrMultiProcessorCount, dev));
    int optin = 0;
    SA_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    ds.smem_optin = (size_t)optin;
    SA_CUDA(cudaFuncSetAttribute(chain_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(chain_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(chain_kernel<false, kWideThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(chain_kernel<false, 384, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(chain_kernel<true, 384, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(chain_kernel<false, kWideThreads, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(rfft_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(rfft_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(irfft_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(irfft_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    {
        cudaFuncAttributes fa;
        SA_CUDA(cudaFuncGetAttributes(&fa, spectral_cta_kernel<8>));
        SA_CUDA(cudaFuncSetAttribute(spectral_cta_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     optin - (int)fa.sharedSizeBytes));
    }
    {
        cudaFuncAttributes fa;
        SA_CUDA(cudaFuncGetAttributes(&fa, spectral_cta_kernel<9>));
        SA_CUDA(cudaFuncSetAttribute(spectral_cta_kernel<9>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     optin - (int)fa.sharedSizeBytes));
    }
    {
        cudaFuncAttributes fa;
        SA_CUDA(cudaFuncGetAttributes(&fa, spectral_cta_kernel<10>));
        SA_CUDA(cudaFuncSetAttribute(spectral_cta_kernel<10>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     optin - (int)fa.sharedSizeBytes));
    }
    {
        cudaFuncAttributes fa;
        SA_CUDA(cudaFuncGetAttributes(&fa, spectral_cta_kernel<11>));
        SA_CUDA(cudaFuncSetAttribute(spectral_cta_kernel<11>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     optin - (int)fa.sharedSizeBytes));
    }
    SA_CUDA(cudaFuncSetAttribute(gather_cta_kernel<kGatherThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(rfft_cta_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(rfft_cta_kernel<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(rfft_cta_kernel<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(rfft_cta_kernel<11>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(irfft_cta_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(irfft_cta_kernel<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(irfft_cta_kernel<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(irfft_cta_kernel<11>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(dct2_cta_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(dct2_cta_kernel<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(dct2_cta_kernel<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(dct2_cta_kernel<11>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(dct3_cta_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(dct3_cta_kernel<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(dct3_cta_kernel<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(dct3_cta_kernel<11>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(spectrum_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(spectrum_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(dct_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(dct_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(dtw_batch_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(dtw_batch_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(dtw_path_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaFuncSetAttribute(dtw_path_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    SA_CUDA(cudaSetDevice(prev));
    ds.ready = true;
    return SA_OK;
}

int ensure_device(int* dev_out) {
    int dev;
    int rc = current_device(&dev);
    if (rc) return rc;
    rc = init_device(dev);
    if (rc) return rc;
    *dev_out = dev;
    return SA_OK;
}

// exp(-2 pi i k / L), k < L, correctly rounded via long double.
int get_twiddles(int dev, int L, const double2** out) {
    std::lock_guard<std::mutex> lk(g_mu);
    DeviceState& ds = dev_state(dev);
    auto it = ds.twiddles.find(L);
    if (it != ds.twiddles.end()) {
        *out = it->second;
        return SA_OK;
    }
    std::vector<double2> h((size_t)L);
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int k = 0; k < L; ++k) {
        long double a = -2.0L * pi * (long double)k / (long double)L;
        h[(size_t)k] = make_double2((double)cosl(a), (double)sinl(a));
    }
    double2* d = nullptr;
    SA_CUDA(cudaMalloc(&d, sizeof(double2) * (size_t)L));
    SA_CUDA(cudaMemcpy(d, h.data(), sizeof(double2) * (size_t)L, cudaMemcpyHostToDevice));
    ds.twiddles[L] = d;
    *out = d;
    return SA_OK;
}

// Pass plan of the complex transform used for a real length L: N = L/2
// (packed) for even L, N = L for odd L; radix 8/4/2 passes first, then one
// generic pass per remaining prime factor (ascending).
int env_int(const char* k, int d);

// allow16: the plan may use radix-16 passes (the standalone transform
// kernels; the chain kernel has no register room for them)
bool make_fft_geo(int64_t L, FftGeo* g, bool allow16 = false, int64_t odd_min = 0) {
    std::memset(g, 0, sizeof(*g));
    if (L < 1) return false;
    g->packed = (L % 2 == 0) ? 1 : 0;
    int64_t N = g->packed ? L / 2 : L;
    g->N = (int32_t)N;
    int64_t rem = N;
    int np = 0;
    int64_t p2 = 1;
    while (rem % 2 == 0) { rem /= 2; p2 *= 2; }
    // power-of-two part: radix-8 passes, except that a final radix-16 pass
    // replaces two passes when log2 is not a multiple of 3 (1024 = 8*8*16
    // instead of 8*8*4*4); radix 16 never runs first (its pass-0 stores would
    // conflict 16 ways in shared memory)
    int lg2 = 0;
    while ((1ll << lg2) < p2) ++lg2;
    const bool use16 = allow16 && env_int("SA_FFT_RADIX16", 1) && lg2 >= 7 && lg2 != 8 && lg2 % 3 != 0;
    int64_t left = use16 ? p2 / 16 : p2;
    while (left > 1) {
        int r = (left >= 8 && left != 16) ? 8 : (left >= 4 ? 4 : 2);
        if (use16 && left == 16) r = 16;  // two radix-16 passes for lg2 % 3 == 2
        if (np >= SA_FFT_MAXPASS) return false;
        g->radix[np++] = (int16_t)r;
        left /= r;
    }
    if (use16) {
        if (np >= SA_FFT_MAXPASS) return false;
        g->radix[np++] = 16;
    }
    for (int64_t f = 3; rem > 1; f += 2) {
        while (rem % f == 0) {
            if (np >= SA_FFT_MAXPASS || f > 32767) return false;
            g->radix[np++] = (int16_t)f;
            rem /= f;
        }
        if (f * f > rem && rem > 1) {
            if (np >= SA_FFT_MAXPASS || rem > 32767) return false;
            g->radix[np++] = (int16_t)rem;
            rem = 1;
        }
    }
    g->npass = np;
    // Large prime factors: the generic passes cost ~N * sum(p) complex MACs;
    // Bluestein costs ~three M-point power-of-two FFTs.  Switch when that is
    // clearly cheaper: its 2M-point buffers cost occupancy, so a margin of
    // 1.8x (measured on the sweep: prime 541 2.1x faster with Bluestein,
    // 909 = 9 * 101 and 1068 = 12 * 89 faster without).
    int64_t gen = 0;
    for (int q = 0; q < np; ++q)
        if (g->radix[q] != 2 && g->radix[q] != 4 && g->radix[q] != 8) gen += N * (int64_t)g->radix[q];
    // odd composite L: the paired-column real transform (sa_fft.cuh rfft_any)
    // runs the last, largest-radix pass on half the columns and the earlier
    // ones on (P + 1) / 2P of the points
    const bool oddon = !g->packed && L >= odd_min && env_int("SA_ODDREAL", 1);
    const bool oddreal = oddon && np >= 2;
    if (oddreal) gen = (gen * 11) / 20;
    if (gen > 0 && env_int("SA_BLUESTEIN", 1)) {
        // odd L (oddon): the real transform needs the bins k <= (N - 1) / 2
        // only, so the circular convolution may wrap the kernel's positive
        // range above (N - 1) / 2: M >= (3N - 1) / 2 instead of 2N - 1 (the
        // inverse runs the same forward transform, irfft_any)
        const int64_t span = oddon ? (3 * N - 1) / 2 : 2 * N - 1;
        int64_t M = 1;
        while (M < span) M <<= 1;
        int lg = 0;
        while ((1ll << lg) < M) ++lg;
        const double blu = 4.5 * (double)M * (double)lg;
        if ((double)gen > 0.1 * env_int("SA_BLUE_X10", 18) * blu || env_int("SA_BLUESTEIN", 1) == 2) {
            if (M > (1ll << 26)) return false;
            g->blue = 1;
            g->M = (int32_t)M;
            int mp = 0;
            for (int64_t left = M; left > 1;) {
                const int r = (left >= 8 && left != 16) ? 8 : (left >= 4 ? 4 : 2);
                g->mradix[mp++] = (int16_t)r;
                left /= r;
            }
            g->mpass = mp;
        }
    }
    // 1: paired columns; 2: Bluestein on the half range of bins
    g->oddreal = g->blue ? (oddon ? 2 : 0) : (oddreal ? 1 : 0);
    return true;
}

// Bluestein tables per (device, N): chirp c[n] = exp(-i pi n^2 / N) (n^2
// reduced mod 2N exactly) and FFT_M of the circular kernel conj(c[|m|]),
// both computed in long double on the host.
std::map<std::pair<int, int>, std::pair<double2*, double2*>> g_blue;

void fft_ld(std::vector<long double>& re, std::vector<long double>& im) {  // in place, radix 2, forward
    const size_t n = re.size();
    for (size_t i = 1, j = 0; i < n; ++i) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) {
            std::swap(re[i], re[j]);
            std::swap(im[i], im[j]);
        }
    }
    const long double pi = 3.141592653589793238462643383279502884L;
    for (size_t len = 2; len <= n; len <<= 1) {
        for (size_t k = 0; k < len / 2; ++k) {
            const long double a = -2.0L * pi * (long double)k / (long double)len;
            const long double wr = cosl(a), wi = sinl(a);
            for (size_t i = k; i < n; i += len) {
                const size_t j = i + len / 2;
                const long double tr = re[j] * wr - im[j] * wi, ti = re[j] * wi + im[j] * wr;
                re[j] = re[i] - tr;
                im[j] = im[i] - ti;
                re[i] += tr;
                im[i] += ti;
            }
        }
    }
}

int finish_geo(int dev, FftGeo* g) {
    if (!g->blue) return SA_OK;
    int rc = get_twiddles(dev, g->M, &g->twM);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(g_mu);
    const bool half = g->oddreal == 2;  // kernel indices -(N - 1) .. (N - 1) / 2 only
    auto key = std::make_pair(dev, half ? -g->N : g->N);
    auto it = g_blue.find(key);
    if (it == g_blue.end()) {
        const int64_t N = g->N, M = g->M;
        const long double pi = 3.141592653589793238462643383279502884L;
        std::vector<double2> ch((size_t)N);
        std::vector<long double> hr((size_t)M, 0.0L), hi((size_t)M, 0.0L);
        for (int64_t n = 0; n < N; ++n) {
            const int64_t q = (int64_t)(((unsigned __int128)n * (unsigned __int128)n) % (unsigned __int128)(2 * N));
            const long double a = -pi * (long double)q / (long double)N;
            const long double c = cosl(a), sn = sinl(a);
            ch[(size_t)n] = make_double2((double)c, (double)sn);
            if (!half || 2 * n <= N - 1) {
                hr[(size_t)n] = c;  // conj(c[n])
                hi[(size_t)n] = -sn;
            }
            if (n > 0) {
                hr[(size_t)(M - n)] = c;
                hi[(size_t)(M - n)] = -sn;
            }
        }
        fft_ld(hr, hi);
        std::vector<double2> bf((size_t)M);
        for (int64_t k = 0; k < M; ++k) bf[(size_t)k] = make_double2((double)hr[(size_t)k], (double)hi[(size_t)k]);
        double2 *dc = nullptr, *db = nullptr;
        SA_CUDA(cudaMalloc(&dc, sizeof(double2) * (size_t)N));
        SA_CUDA(cudaMalloc(&db, sizeof(double2) * (size_t)M));
        SA_CUDA(cudaMemcpy(dc, ch.data(), sizeof(double2) * (size_t)N, cudaMemcpyHostToDevice));
        SA_CUDA(cudaMemcpy(db, bf.data(), sizeof(double2) * (size_t)M, cudaMemcpyHostToDevice));
        it = g_blue.emplace(key, std::make_pair(dc, db)).first;
    }
    g->chirp = it->second.first;
    g->bfft = it->second.second;
    return SA_OK;
}


std::map<std::pair<int, int>, double2*> g_dct_tw;  // (device, N) -> exp(-i pi k / 2N)

int get_dct_twiddles(int dev, int N, const double2** out) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto key = std::make_pair(dev, N);
    auto it = g_dct_tw.find(key);
    if (it != g_dct_tw.end()) {
        *out = it->second;
        return SA_OK;
    }
    std::vector<double2> h((size_t)N);
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int k = 0; k < N; ++k) {
        long double a = -pi * (long double)k / (2.0L * (long double)N);
        h[(size_t)k] = make_double2((double)cosl(a), (double)sinl(a));
    }
    double2* d = nullptr;
    SA_CUDA(cudaMalloc(&d, sizeof(double2) * (size_t)N));
    SA_CUDA(cudaMemcpy(d, h.data(), sizeof(double2) * (size_t)N, cudaMemcpyHostToDevice));
    g_dct_tw[key] = d;
    *out = d;
    return SA_OK;
}

// doubles per buffer a spectral stage needs at length L
// doubles per row buffer for an L-point real transform (Bluestein: M complex)
int64_t fft_lcap(int64_t L, const FftGeo* g = nullptr) {
    if (g && g->oddreal == 1) {
        // paired-column real transform of L = P q: (P + 1) / 2 * q complex
        // points through the first passes, P * (q + 1) / 2 into the last
        const int64_t P = g->radix[g->npass - 1], q = L / P;
        return L + std::max(P, q) + 2;
    }
    const int64_t base = (L % 2 == 0) ? L + 2 : 2 * L + 2;
    return (g && g->blue) ? std::max<int64_t>(base, 2 * (int64_t)g->M + 2) : base;
}

bool is_spectral(int op) { return op == SA_OP_APP || op == SA_OP_FREQ_MASK || op == SA_OP_SINUSOID; }

struct Plan {
    ChainParams p;
    Layout lay;
    int grid;
    bool wide = false;  // short series: chain_kernel<false, kWideThreads>
    bool odd = false;   // some spectral stage has a non-power-of-two FFT plan: chain_kernel<*, *, true>
    int warps;     // warps (= series in flight) per CTA
    size_t smem;   // dynamic smem per CTA
    bool global = false;  // row buffers in a global scratch of grid * warps slots
};

int env_int(const char* k, int d) {
    const char* v = getenv(k);
    return v && *v ? atoi(v) : d;
}

// Relative per-series cost of an operator at L ~ 1e3 (tools/op_timing.py),
// used only to choose which gates form the scheduling key.
double op_cost(int op) {
    switch (op) {
        case SA_OP_APP: return 10.0;
        case SA_OP_FREQ_MASK: case SA_OP_SINUSOID: return 4.5;
        case SA_OP_JITTER: case SA_OP_NOISE_GAUSSIAN: case SA_OP_NOISE_SPIKE: return 3.0;
        case SA_OP_SPEED_WARP: case SA_OP_DRIFT: case SA_OP_TIME_WARP: return 2.4;
        case SA_OP_CONVOLVE: case SA_OP_RESIZE: return 1.5;
        case SA_OP_NOISE_UNIFORM: case SA_OP_WINDOW_WARP: case SA_OP_DROPOUT: return 1.0;
        case SA_OP_QUANTIZE: case SA_OP_POOL: return 0.5;
        default: return 0.1;
    }
}

// Lower the ABI stage table into kernel parameters and a launch shape.
// spread: the caller waits for this launch alone (synchronous entry points),
// so a batch of less than one wave is spread over the SMs for latency; the
// asynchronous launch keeps full CTAs (concurrent streams fill the rest).
int make_plan(int dev, const sa_stage* stages, int32_t ns, const double* aux, int32_t n_aux, uint64_t seed,
              int64_t offset, int64_t n, int64_t len_in, int64_t len_out, Plan* plan, bool spread = false) {
    if (ns < 0 || ns > SA_MAX_STAGES) return fail(SA_ERR_INVALID_ARG, "n_stages out of range");
    if (n_aux < 0 || n_aux > SA_MAX_AUX) return fail(SA_ERR_INVALID_ARG, "aux table too large");
    if (n < 0 || len_in < 1 || len_out < 1) return fail(SA_ERR_INVALID_ARG, "bad batch shape");
    if (len_in > (1 << 24)) return fail(SA_ERR_UNSUPPORTED, "series longer than 2^24");
    ChainParams& p = plan->p;
    std::memset(&p, 0, sizeof(p));
    p.ns = ns;
    p.repeat_r = 1;
    p.seed = seed;
    p.offset = offset;
    p.len_in = (int32_t)len_in;
    p.len_out = (int32_t)len_out;
    if (n_aux) std::memcpy(p.aux, aux, sizeof(double) * (size_t)n_aux);
    int64_t L = len_in, lmax = len_in;
    int small = 64, iscr = 16;
    int64_t spike_lcap = 0;
    bool after_repeat = false;
    for (int j = 0; j < ns; ++j) {
        const sa_stage& s = stages[j];
        DevStage& d = p.st[j];
        if (s.op < 1 || s.op >= SA_OP_MAX) return fail(SA_ERR_INVALID_ARG, "unknown op code");
        d.op = s.op;
        d.index = s.index;
        d.prob = s.probability;
        for (int k = 0; k < 4; ++k) {
            d.f[k] = s.f[k];
            d.i[k] = s.i[k];
        }
        d.aux_off = s.aux_off;
        d.aux_len = s.aux_len;
        d.post_repeat = after_repeat ? 1 : 0;
        d.len_in = (int32_t)L;
        if (s.op == SA_OP_REPEAT && s.probability != 0.0 && s.i[0] != 1) {
            if (p.repeat_r != 1) return fail(SA_ERR_INVALID_ARG, "at most one repeat stage");
            p.repeat_r = (int32_t)s.i[0];
            after_repeat = true;
        }
        if (s.op == SA_OP_CONVOLVE && (s.aux_off < 0 || s.aux_len < 1 || s.aux_off + s.aux_len > n_aux))
            return fail(SA_ERR_INVALID_ARG, "convolve taps out of range");
        if (is_spectral(s.op) && s.probability > 0.0) {
            if (!make_fft_geo(L, &d.fft, false, env_int("SA_ODDREAL_MIN", 0)))
                return fail(SA_ERR_UNSUPPORTED, "no FFT plan for length " + std::to_string(L));
            // anything but a plain radix-8/4/2 plan runs the ODD instantiations
            bool plain = !d.fft.blue && !d.fft.oddreal;
            for (int q = 0; q < d.fft.npass; ++q)
                plain = plain && (d.fft.radix[q] == 2 || d.fft.radix[q] == 4 || d.fft.radix[q] == 8);
            plan->odd = plan->odd || !plain;
            int rc = get_twiddles(dev, (int)L, &d.tw);
            if (!rc) rc = finish_geo(dev, &d.fft);
            if (rc) return rc;
            spike_lcap = std::max<int64_t>(spike_lcap, fft_lcap(L, &d.fft));
        }
        if (s.probability == 1.0 && (s.op == SA_OP_CROP || s.op == SA_OP_RESIZE)) L = s.i[0];
        d.len_out = (int32_t)L;
        lmax = std::max(lmax, L);
        // scratch needs
        if (s.op == SA_OP_DRIFT) small = std::max<int>(small, (int)(3 * s.i[0]) + 2);
        if (s.op == SA_OP_TIME_WARP) small = std::max<int>(small, (int)(3 * s.i[0]) + 2);
        if (s.op == SA_OP_WINDOW_WARP) small = std::max<int>(small, (int)(3 * s.i[1]) + 2);
        if (s.op == SA_OP_SPEED_WARP) {
            small = std::max<int>(small, (int)(2 * (s.i[0] + 1)) + 2);
            iscr = std::max<int>(iscr, (int)s.i[0] + 2);
        }
        if (s.op == SA_OP_NOISE_SPIKE) small = std::max<int>(small, 2 * (int)(lmax / 64 + 2) + 8);
        if (s.op == SA_OP_PERMUTE) iscr = std::max<int>(iscr, (int)s.i[0] + 1);
        if (s.op == SA_OP_NOISE_SPIKE) {  // choice scratch lives in the second buffer
            int64_t k = s.i[0];
            uint32_t mask = (uint32_t)(1.2 * (double)k);
            mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4; mask |= mask >> 8; mask |= mask >> 16;
            int64_t need_words = ((L > 10000 && k > L / 50) ? L : (int64_t)mask + 1) + k + 1;
            spike_lcap = std::max<int64_t>(spike_lcap, (need_words + 1) / 2);
        }
    }
    if (L != len_out) return fail(SA_ERR_INVALID_ARG, "len_out does not match the projected length");
    p.rows_out = n * p.repeat_r;
    p.lcap = (int32_t)((std::max<int64_t>(lmax + 2, spike_lcap) + 1) & ~1LL);
    p.small_words = small;
    p.iscr_words = iscr;
    plan->lay = make_layout(p.lcap, ns, small, iscr);
    DeviceState& ds = dev_state(dev);
    // Row buffers in shared memory unless (a) they do not fit, or (b) so few
    // warps fit (<= 3 per SM: long odd lengths, Bluestein buffers) that the
    // SM's four schedulers starve while there are rows for several waves:
    // then the buffers move to global memory (L2 resident), which lets 12
    // warps per SM run (sweep: L = 2369 1.9x, Bluestein 541 / 1707 1.3-2x).
    const size_t smem_fit = (ds.smem_optin - kCtaShared) / std::max<size_t>(plan->lay.total, 1);
    // With 4-5 warps the answer depends on the chain: compute-heavy chains
    // (APP-level work per row) gain 8-16% from 12 warps over the L2-resident
    // scratch, light ones (one Jitter, one TimeWarp) lose 25-130% to its
    // traffic (L = 2300 .. 2900, tools/oddreal_session3.sh).
    double work = 0.0;
    for (int j = 0; j < ns; ++j) work += stages[j].probability * op_cost(stages[j].op);
    // At 6 warps only Bluestein chains gain (their rows run four M-point FFTs
    // per spectral stage: config 5's chain at L = 541 1.83 ms in the scratch
    // against 2.05; the same chain at L = 2136, generic passes, 2.88 against 2.80).
    bool blue = false;
    for (int j = 0; j < ns; ++j) blue = blue || (is_spectral(stages[j].op) && stages[j].probability > 0.0 && p.st[j].fft.blue);
    const int starved_fit = env_int("SA_STARVED_FIT", (work >= 15.0 && blue) ? 6 : (work >= 8.0 ? 5 : 3));
    const bool starved = smem_fit >= 1 && smem_fit <= (size_t)starved_fit && env_int("SA_AUTO_GLOBAL", 1) &&
                         p.rows_out > 3 * (int64_t)ds.sms * (int64_t)smem_fit;
    if (plan->lay.total + kCtaShared > ds.smem_optin || starved || env_int("SA_FORCE_GLOBAL", 0)) {
        // long series: the two row buffers move to global memory (L2 / HBM
        // resident, same code); shared memory keeps the window and scratch
        plan->global = true;
        if (env_int("SA_GLOBAL_ALIGN", 1)) p.lcap = (p.lcap + 15) & ~15;  // 128-byte rows in the scratch
        plan->lay = make_layout(0, ns, small, iscr);
        if (plan->lay.total + kCtaShared > ds.smem_optin)
            return fail(SA_ERR_UNSUPPORTED, "stage scratch too large for shared memory");
    }
    // Stage-major CTAs: `warps` series per CTA walk the chain in lockstep
    // (a barrier every `sync_every` stages) so the SM works through one
    // operator's code at a time (the fused kernel is
    // instruction-fetch bound when warps drift apart).
    const int per_warp = (int)plan->lay.total;
    int fit = (int)((ds.smem_optin - kCtaShared) / (size_t)per_warp);
    int warps = env_int("SA_CTA_WARPS", 0);
    // short series (shared memory holds >= 16 rows): the wide instantiation,
    // 16 warps at 128 registers instead of 12 at 168 -- their rows are
    // latency bound on per-row fixed costs (sweep L = 29 .. 440: -8..15%)
    plan->wide = !plan->global && fit >= kWideThreads / 32 && env_int("SA_WIDE", 1) != 0;
    const int wmax = plan->wide ? kWideThreads / 32 : 12;
    if (warps <= 0) warps = std::min(wmax, std::max(1, fit));
    // less than one wave of rows: spread them over the SMs (a row's chain is
    // latency bound; 38 rows on 4 SMs ran 1.6x slower than on 38)
    if (spread && env_int("SA_CTA_WARPS", 0) <= 0 && p.rows_out < (int64_t)ds.sms * warps)
        warps = (int)std::max<int64_t>(1, (p.rows_out + ds.sms - 1) / ds.sms);
    warps = std::max(1, std::min(warps, std::min(wmax, fit)));
    plan->warps = warps;
    plan->smem = (size_t)per_warp * warps + kCtaShared;
    p.sync_every = ns > 1 ? env_int("SA_SYNC_EVERY", 4) : 0;
    // barrier placement (bit j: barrier before stage j).  Policy 0: every
    // `sync_every` stages; policy 1: before every stage whose operator is
    // expensive (op_cost >= threshold) and every `sync_every` cheap stages.
    p.sync_mask = 0;
    if (p.sync_every) {
        const int policy = env_int("SA_SYNC_POLICY", 0);
        const double thr = env_int("SA_SYNC_COST_X10", 20) / 10.0;
        int since = 0;
        for (int j = 0; j < ns; ++j) {
            bool b;
            if (policy == 1) {
                const bool heavy = op_cost(stages[j].op) >= thr;
                b = heavy || since >= p.sync_every;
                since = heavy ? 0 : since + 1;
                if (b && !heavy) since = 0;
            } else {
                b = (j % p.sync_every) == 0;
            }
            if (b) p.sync_mask |= 1ull << j;
        }
        if (const char* m = getenv("SA_SYNC_MASK")) p.sync_mask = strtoull(m, nullptr, 16) | 1ull;  // experiments
    }
    // scheduling key: gated (0 < p < 1) stages, most expensive first
    {
        std::vector<std::pair<double, int>> cand;
        for (int j = 0; j < ns; ++j)
            if (stages[j].probability > 0.0 && stages[j].probability < 1.0 && stages[j].op != SA_OP_REPEAT)
                cand.push_back({-op_cost(stages[j].op), j});
        std::stable_sort(cand.begin(), cand.end());
        int kb = (int)std::min<size_t>((size_t)std::max(0, std::min(24, env_int("SA_SCHEDULE_BITS", 16))), cand.size());
        // sorted keys put similar fire patterns next to each other even when
        // buckets are sparse; only keep the histogram proportionate
        while (kb > 0 && ((int64_t)1 << kb) > 4 * p.rows_out) --kb;
        // small batches: a few CTAs, three extra launches would cost more than the balance gains
        if (p.rows_out < env_int("SA_SCHEDULE_MIN_ROWS", 4096)) kb = 0;
        if (env_int("SA_SCHEDULE", 1) == 0 || p.rows_out > INT32_MAX) kb = 0;
        p.key_bits = kb;
        for (int q = 0; q < kb; ++q) p.key_stage[q] = (int8_t)cand[q].second;
        // adaptive lockstep compares EVERY gated stage: rows that differ only
        // in cheap stages still drift apart over a row (measured: comparing
        // only the sorted gates costs 3% at 1e6 rows); ~0: always barrier
        p.uni_mask = 0;
        for (size_t q = 0; q < cand.size(); ++q) p.uni_mask |= 1ull << cand[q].second;
        if (!env_int("SA_ADAPTIVE_SYNC", 1)) p.uni_mask = ~0ull;
    }
    int per_sm = 0;
    {
        static std::mutex occ_mu;
        static std::map<std::pair<int, size_t>, int> occ_cache;  // (warps, smem) -> CTAs per SM
        std::lock_guard<std::mutex> lk(occ_mu);
        auto key = std::make_pair(warps * 4 + (plan->global ? 1 : 0) + (plan->wide ? 2 : 0), plan->smem);
        auto it = occ_cache.find(key);
        if (it != occ_cache.end()) {
            per_sm = it->second;
        } else {
            cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &per_sm,
                plan->odd ? (plan->global ? chain_kernel<true, 384, true>
                                          : (plan->wide ? chain_kernel<false, kWideThreads, true> : chain_kernel<false, 384, true>))
                          : (plan->global ? chain_kernel<true>
                                          : (plan->wide ? chain_kernel<false, kWideThreads> : chain_kernel<false>)),
                32 * warps, plan->smem);
            if (e != cudaSuccess) return cuda_fail(e, "occupancy");
            occ_cache[key] = per_sm;
        }
    }
    per_sm = std::max(per_sm, 1);
    int64_t ctas_needed = (p.rows_out + warps - 1) / warps;
    int64_t want = (int64_t)ds.sms * per_sm;
    if (plan->global) {  // bound the scratch: <= 4 GB of row buffers in flight
        const int64_t slot_b = 16 * (int64_t)p.lcap;
        const int64_t slots = std::max<int64_t>(1, (4ll << 30) / slot_b);
        want = std::min<int64_t>(want, std::max<int64_t>(1, slots / warps));
        if (slots < warps) {
            plan->warps = warps = (int)slots;
            plan->smem = (size_t)per_warp * warps + kCtaShared;
            ctas_needed = (p.rows_out + warps - 1) / warps;
        }
    }
    plan->grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, ctas_needed));
    return SA_OK;
}

// Schedule (fire-pattern counting sort) and launch the chain kernel for the
// rows described by plan->p (in/out/flags/offset/rows_out already set).
// stream-ordered scratch freed on every return path
struct StreamScratch {
    cudaStream_t st;
    std::vector<void*> ptrs;
    explicit StreamScratch(cudaStream_t s) : st(s) {}
    template <class T>
    cudaError_t alloc(T** p, size_t bytes) {
        cudaError_t e = sa_malloc_async((void**)p, bytes, st);
        if (e == cudaSuccess) ptrs.push_back(*p);
        return e;
    }
    ~StreamScratch() {
        for (void* q : ptrs) cudaFreeAsync(q, st);
    }
};

bool cta_fft_len(int64_t L, std::initializer_list<const void*> aligned16);
int cta_launch_shape(int dev, const void* kern, int64_t L, int64_t n, int* threads, size_t* smem, int* grid);

// Spectral-only chain on the CTA FFT (spectral_cta_kernel): every stage a
// FrequencyMask / RandomSinusoid, length L = 2N with N = 256 .. 2048 a power
// of two, no Repeat, rows 16-byte aligned.  Returns the W_L table or null.
const double2* spectral_cta_table(const Plan* plan) {
    const ChainParams& p = plan->p;
    const int64_t L = p.len_in;
    if (plan->global || p.repeat_r != 1 || p.len_out != L || p.ns < 1 || p.ns > 64 ||
        env_int("SA_CTA_CHAIN", 1) == 0 || !cta_fft_len(L, {p.in, p.out}))
        return nullptr;
    const double2* tw = nullptr;
    for (int j = 0; j < p.ns; ++j) {
        if (p.st[j].op != SA_OP_FREQ_MASK && p.st[j].op != SA_OP_SINUSOID) return nullptr;
        if (p.st[j].tw) tw = p.st[j].tw;
    }
    return tw;
}

// Gather-only chain on a CTA per row (gather_cta_kernel): every stage a
// SpeedWarp (n_speed_change <= 7), Resize, Convolve, Rotate or Reverse, no
// Repeat, both row buffers in shared memory.  Returns its dynamic smem or 0.
size_t gather_cta_smem(const Plan* plan) {
    const ChainParams& p = plan->p;
    if (plan->global || p.repeat_r != 1 || p.ns < 1 || p.ns > 64 || env_int("SA_GATHER_CTA", 1) == 0) return 0;
    for (int j = 0; j < p.ns; ++j) {
        const DevStage& st = p.st[j];
        switch (st.op) {
            case SA_OP_SPEED_WARP:
                if (st.i[0] > kGatherMaxSpeeds - 1) return 0;
                break;
            case SA_OP_RESIZE: case SA_OP_CONVOLVE: case SA_OP_ROTATE: case SA_OP_REVERSE: break;
            default: return 0;
        }
    }
    const size_t smem = 16 * (size_t)p.lcap + 8 * (kGatherMaxSpeeds + 2) + 4 * (kGatherMaxSpeeds + 8) +
                        sizeof(GatherDraw) * (size_t)p.ns;
    return smem <= dev_state(current_device_id()).smem_optin ? smem : 0;
}

int launch_chain(Plan* plan, cudaStream_t stream) {
    ChainParams& p = plan->p;
    if (p.rows_out == 0) return SA_OK;
    if (const size_t gsm = gather_cta_smem(plan)) {
        DeviceState& dsg = dev_state(current_device_id());
        int per_sm = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gather_cta_kernel<kGatherThreads>,
                                                                      kGatherThreads, gsm);
        if (e != cudaSuccess) return cuda_fail(e, "occupancy");
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)dsg.sms * std::max(per_sm, 1), p.rows_out));
        p.order = nullptr;
        StreamScratch scr(stream);
        GatherDraw* draws;
        SA_CUDA(scr.alloc(&draws, sizeof(GatherDraw) * (size_t)(p.rows_out * p.ns)));
        const int gd = (int)std::min<int64_t>((int64_t)dsg.sms * 8, (p.rows_out * p.ns + 255) / 256);
        gather_draw_kernel<<<gd, 256, 0, stream>>>(p, draws);
        gather_cta_kernel<kGatherThreads><<<grid, kGatherThreads, gsm, stream>>>(p, draws);
        SA_CUDA(cudaGetLastError());
        __atomic_add_fetch(&g_launches, 2, __ATOMIC_RELAXED);
        return SA_OK;
    }
    if (const double2* tw = spectral_cta_table(plan)) {
        const int64_t N = p.len_in / 2;
        const void* kern = N == 256 ? (const void*)spectral_cta_kernel<8>
                         : N == 512 ? (const void*)spectral_cta_kernel<9>
                         : N == 1024 ? (const void*)spectral_cta_kernel<10> : (const void*)spectral_cta_kernel<11>;
        int threads, grid;
        size_t smem;
        int rc = cta_launch_shape(current_device_id(), kern, p.len_in, p.rows_out, &threads, &smem, &grid);
        if (rc) return rc;
        p.order = nullptr;
        DeviceState& dsc = dev_state(current_device_id());
        StreamScratch scr(stream);
        SpecDraw* draws;
        SA_CUDA(scr.alloc(&draws, sizeof(SpecDraw) * (size_t)(p.rows_out * p.ns)));
        const int gd = (int)std::min<int64_t>((int64_t)dsc.sms * 8, (p.rows_out * p.ns + 255) / 256);
        spectral_draw_kernel<<<gd, 256, 0, stream>>>(p, draws);
        void* args[] = {&p, (void*)&tw, (void*)&draws};
        SA_CUDA(cudaLaunchKernel(kern, dim3(grid), dim3(threads), args, smem, stream));
        __atomic_add_fetch(&g_launches, 2, __ATOMIC_RELAXED);
        return SA_OK;
    }
    DeviceState& ds = dev_state(current_device_id());
    StreamScratch scratch(stream);
    p.order = nullptr;
    while (p.key_bits > 0 && ((int64_t)1 << p.key_bits) > 4 * p.rows_out) --p.key_bits;
    if (p.key_bits > 0) {
        const int nb = 1 << p.key_bits;
        uint32_t *keys, *hist;
        int32_t* order;
        SA_CUDA(scratch.alloc(&keys, sizeof(uint32_t) * (size_t)p.rows_out));
        SA_CUDA(scratch.alloc(&hist, sizeof(uint32_t) * (size_t)nb));
        SA_CUDA(scratch.alloc(&order, sizeof(int32_t) * (size_t)p.rows_out));
        SA_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (size_t)nb, stream));
        const int g = (int)std::min<int64_t>((int64_t)ds.sms * 8, (p.rows_out + 255) / 256);
        key_hist_kernel<<<g, 256, 0, stream>>>(p, keys, hist);
        key_scan_kernel<<<1, 1024, 0, stream>>>(hist, nb);
        key_scatter_kernel<<<g, 256, 0, stream>>>(p.rows_out, keys, hist, order);
        SA_CUDA(cudaGetLastError());
        __atomic_add_fetch(&g_launches, 3, __ATOMIC_RELAXED);
        p.order = order;
    }
    if (plan->global) {
        SA_CUDA(scratch.alloc(&p.gbuf, sizeof(double) * 2 * (size_t)p.lcap * (size_t)plan->grid * plan->warps));
        p.bulk_in = 0;  // TMA bulk copies target shared memory only
    }
    if (plan->odd && plan->global) chain_kernel<true, 384, true><<<plan->grid, 32 * plan->warps, plan->smem, stream>>>(p);
    else if (plan->odd && plan->wide) chain_kernel<false, kWideThreads, true><<<plan->grid, 32 * plan->warps, plan->smem, stream>>>(p);
    else if (plan->odd) chain_kernel<false, 384, true><<<plan->grid, 32 * plan->warps, plan->smem, stream>>>(p);
    else if (plan->global) chain_kernel<true><<<plan->grid, 32 * plan->warps, plan->smem, stream>>>(p);
    else if (plan->wide) chain_kernel<false, kWideThreads><<<plan->grid, 32 * plan->warps, plan->smem, stream>>>(p);
    else chain_kernel<false><<<plan->grid, 32 * plan->warps, plan->smem, stream>>>(p);
    SA_CUDA(cudaGetLastError());
    __atomic_add_fetch(&g_launches, 1, __ATOMIC_RELAXED);
    return SA_OK;
}

int launch_plan(Plan* plan, const double* d_in, double* d_out, uint32_t* d_flags, cudaStream_t stream) {
    ChainParams& p = plan->p;
    p.in = d_in;
    p.out = d_out;
    p.flags = d_flags;
    p.bulk_in = ((p.len_in & 1) == 0 && (reinterpret_cast<uintptr_t>(d_in) & 15u) == 0) ? 1 : 0;
    SA_CUDA(cudaMemsetAsync(d_flags, 0, sizeof(uint32_t), stream));
    return launch_chain(plan, stream);
}

int flags_status(uint32_t f) {
    if (f & SA_FLAG_WARP_MONOTONE) return fail(SA_ERR_WARP_MONOTONE, "warp map failed to stay strictly increasing");
    if (f & SA_FLAG_NONFINITE) return fail(SA_ERR_NONFINITE, "batch contains non-finite values (NaN or Inf)");
    return SA_OK;
}

// Buffers of the one-warp transform kernels: 2 * lcap doubles + a Philox
// window per CTA in shared memory; when that does not fit, the row buffers
// go to a global scratch of grid slots (<= 4 GB) and only the window stays.
int fft_plan_smem(int dev, int64_t L, int* lcap, size_t* smem, int* grid, const void* kern, int64_t n,
                  bool* global, const FftGeo* geo = nullptr) {
    *lcap = (int)((fft_lcap(L, geo) + 1) & ~1LL);
    *smem = (size_t)(*lcap) * 8 * 2 + 8 * SA_WIN + 64;
    DeviceState& ds = dev_state(dev);
    *global = *smem > ds.smem_optin || env_int("SA_FORCE_GLOBAL", 0) != 0;
    if (*global) *smem = 8 * SA_WIN + 64 + 32;
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32, *smem);
    if (e != cudaSuccess) return cuda_fail(e, "occupancy");
    int64_t g = (int64_t)ds.sms * std::max(per_sm, 1);
    if (*global) g = std::min<int64_t>(g, std::max<int64_t>(1, (4ll << 30) / (16 * (int64_t)*lcap)));
    *grid = (int)std::max<int64_t>(1, std::min<int64_t>(g, n));
    return SA_OK;
}

// CTA transform path: even length, power-of-two complex length N = L / 2
// in [256, 2048] (SA_CTA_FFT=0 disables).  T = N / 8 threads, 16 N bytes.
bool cta_fft_len(int64_t L, std::initializer_list<const void*> aligned16) {
    const int64_t N = L / 2;
    for (const void* q : aligned16)  // 16-byte row accesses (cp.async / double2 stores)
        if (reinterpret_cast<uintptr_t>(q) & 15) return false;
    return (L % 2 == 0) && N >= 256 && N <= 2048 && (N & (N - 1)) == 0 && env_int("SA_CTA_FFT", 1) != 0;
}
// kernel instantiation for N = L / 2 = 2^lg (8 <= lg <= 11)
#define SA_CTA_PICK(kern)                                                     \
    inline const void* pick_##kern(int64_t L) {                               \
        switch (L / 2) {                                                      \
            case 256: return (const void*)kern<8>;                            \
            case 512: return (const void*)kern<9>;                            \
            case 1024: return (const void*)kern<10>;                          \
            default: return (const void*)kern<11>;                            \
        }                                                                     \
    }
SA_CTA_PICK(rfft_cta_kernel)
SA_CTA_PICK(irfft_cta_kernel)
SA_CTA_PICK(dct2_cta_kernel)
SA_CTA_PICK(dct3_cta_kernel)

int cta_launch(const void* kern, int grid, int threads, size_t smem, cudaStream_t st, FftParams& p) {
    void* args[] = {&p};
    SA_CUDA(cudaLaunchKernel(kern, dim3(grid), dim3(threads), args, smem, st));
    __atomic_add_fetch(&g_launches, 1, __ATOMIC_RELAXED);
    return SA_OK;
}

int cta_launch_shape(int dev, const void* kern, int64_t L, int64_t n, int* threads, size_t* smem, int* grid) {
    const int64_t N = L / 2;
    *threads = (int)(N / 8);
    *smem = 16 * (size_t)(2 * N + 1);
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, *threads, *smem);
    if (e != cudaSuccess) return cuda_fail(e, "occupancy");
    const int64_t g = (int64_t)dev_state(dev).sms * std::max(per_sm, 1);
    *grid = (int)std::max<int64_t>(1, std::min<int64_t>(g, n));
    return SA_OK;
}

// global scratch for a transform launch (freed stream-ordered by the caller)
int alloc_row_bufs(bool global, int lcap, int grid, cudaStream_t st, double** out) {
    *out = nullptr;
    if (!global) return SA_OK;
    SA_CUDA(sa_malloc_async((void**)out, sizeof(double) * 2 * (size_t)lcap * (size_t)grid, st));
    return SA_OK;
}

#include "sa_host_stage.inc"

// argument checks of the C ABI, before any device work
#define SA_REQUIRE(cond, what)                                           \
    do {                                                                 \
        if (!(cond)) return fail(SA_ERR_INVALID_ARG, std::string(what)); \
    } while (0)

}  // namespace

// ====================================================================== C ABI
extern "C" {

int sa_abi_version(void) { return SA_ABI_VERSION; }

const char* sa_last_error(void) { return g_err.c_str(); }

int64_t sa_launch_count(void) { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

int sa_init(int32_t device) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) return fail(SA_ERR_NO_DEVICE, "no CUDA device available");
    if (device < 0 || device >= count || device >= kMaxDevices)
        return fail(SA_ERR_INVALID_ARG, "device index out of range");
    SA_CUDA(cudaSetDevice(device));
    return init_device(device);
}

int sa_derive_key(uint64_t seed, uint64_t j, uint64_t i, uint64_t* lo, uint64_t* hi) {
    SA_REQUIRE(lo && hi, "sa_derive_key: null output");
    auto mix = [](uint64_t z) {
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    };
    uint64_t s = mix(seed);
    s = mix(s + kGolden + j);
    s = mix(s + kGolden + i);
    *lo = mix(s);
    *hi = mix(s + kGolden);
    return SA_OK;
}

int sa_pipeline_launch(const sa_stage* stages, int32_t n_stages, const double* aux, int32_t n_aux,
                       uint64_t master_seed, int64_t series_offset, const double* d_in, int64_t n,
                       int64_t len_in, double* d_out, int64_t len_out, uint32_t* d_flags, void* stream) {
    SA_REQUIRE(n_stages >= 0 && (n_stages == 0 || stages), "stage table missing");
    SA_REQUIRE(n_aux >= 0 && (n_aux == 0 || aux), "aux table missing");
    SA_REQUIRE(n >= 0 && len_in >= 1 && len_out >= 1, "bad batch shape");
    SA_REQUIRE(n == 0 || (d_in && d_out), "null batch buffer");
    SA_REQUIRE(d_flags, "null flag word");
    int dev;
    int rc = ensure_device(&dev);
    if (rc) return rc;
    Plan plan;
    rc = make_plan(dev, stages, n_stages, aux, n_aux, master_seed, series_offset, n, len_in, len_out, &plan);
    if (rc) return rc;
    return launch_plan(&plan, d_in, d_out, d_flags, (cudaStream_t)stream);
}

int sa_pipeline_run(const sa_stage* stages, int32_t n_stages, const double* aux, int32_t n_aux,
                    uint64_t master_seed, int64_t series_offset, const double* d_in, int64_t n, int64_t len_in,
                    double* d_out, int64_t len_out, void* stream) {
    SA_REQUIRE(n_stages >= 0 && (n_stages == 0 || stages), "stage table missing");
    SA_REQUIRE(n_aux >= 0 && (n_aux == 0 || aux), "aux table missing");
    SA_REQUIRE(n >= 0 && len_in >= 1 && len_out >= 1, "bad batch shape");
    SA_REQUIRE(n == 0 || (d_in && d_out), "null batch buffer");
    int dev;
    int rc = ensure_device(&dev);
    if (rc) return rc;
    Plan plan;
    rc = make_plan(dev, stages, n_stages, aux, n_aux, master_seed, series_offset, n, len_in, len_out, &plan, true);
    if (rc) return rc;
    uint32_t* dflag = nullptr;
    SA_CUDA(sa_malloc_async((void**)&dflag, sizeof(uint32_t), (cudaStream_t)stream));
    rc = launch_plan(&plan, d_in, d_out, dflag, (cudaStream_t)stream);
    if (rc) return rc;
    uint32_t h = 0;
    SA_CUDA(cudaMemcpyAsync(&h, dflag, sizeof(uint32_t), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    SA_CUDA(cudaFreeAsync(dflag, (cudaStream_t)stream));
    SA_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    return flags_status(h);
}

int sa_pipeline_run_host(const sa_stage* stages, int32_t n_stages, const double* aux, int32_t n_aux,
                         uint64_t master_seed, int64_t series_offset, const double* h_in, int64_t n,
                         int64_t len_in, double* h_out, int64_t len_out) {
    SA_REQUIRE(n_stages >= 0 && (n_stages == 0 || stages), "stage table missing");
    SA_REQUIRE(n_aux >= 0 && (n_aux == 0 || aux), "aux table missing");
    SA_REQUIRE(n >= 0 && len_in >= 1 && len_out >= 1, "bad batch shape");
    SA_REQUIRE(n == 0 || (h_in && h_out), "null batch buffer");
    int dev;
    int rc = ensure_device(&dev);
    if (rc) return rc;
    Plan plan;
    rc = make_plan(dev, stages, n_stages, aux, n_aux, master_seed, series_offset, n, len_in, len_out, &plan, true);
    if (rc) return rc;
    const int64_t r = plan.p.repeat_r;
    std::lock_guard<std::mutex> lk(g_host_mu[dev < 0 ? 0 : (dev >= kMaxDevices ? kMaxDevices - 1 : dev)]);
    DeviceState& ds = dev_state(dev);
    // chunks of rows through the host-staging runtime (sa_host_stage.inc);
    // each slot accumulates the kernel's status bits in its own flag word
    const HostIn in{h_in, 8 * len_in};
    const HostOut out{h_out, 8 * len_out * r};
    if ((rc = ensure_streams(ds))) return rc;
    for (int k = 0; k < DeviceState::NS; ++k)  // ordered before each slot's kernels
        SA_CUDA(cudaMemsetAsync(ds.dflags + k, 0, sizeof(uint32_t), ds.hs[k]));
    rc = run_rows_host(dev, n, &in, 1, &out, 1,
                       [&](int k, int64_t r0, int64_t rows, const void* const* d_in, void* const* d_out,
                           cudaStream_t st) -> int {
                           Plan pl = plan;
                           pl.p.offset = series_offset + r0;
                           pl.p.rows_out = rows * r;
                           pl.grid = (int)std::max<int64_t>(
                               1, std::min<int64_t>(plan.grid, (pl.p.rows_out + plan.warps - 1) / plan.warps));
                           pl.p.in = (const double*)d_in[0];
                           pl.p.out = (double*)d_out[0];
                           pl.p.flags = ds.dflags + k;
                           pl.p.bulk_in = ((len_in & 1) == 0) ? 1 : 0;
                           return launch_chain(&pl, st);
                       });
    if (rc) return rc;
    // every slot's flag reset (and kernels) must be complete before the read:
    // run_rows_host only waits on the slots that received rows, and the slot
    // streams are non-blocking (not ordered with the legacy stream)
    for (int k = 0; k < DeviceState::NS; ++k) SA_CUDA(cudaStreamSynchronize(ds.hs[k]));
    uint32_t hflags[DeviceState::NS] = {0, 0, 0};
    SA_CUDA(cudaMemcpy(hflags, ds.dflags, DeviceState::NS * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    uint32_t f = 0;
    for (int k = 0; k < DeviceState::NS; ++k) f |= hflags[k];
    return flags_status(f);
}

// Row-wise transforms over host buffers (the reference API's numpy arrays):
// the host-staging runtime around the device entry points below.
static int host_rows(int64_t n, const HostIn* ins, int nin, const HostOut* outs, int nout,
                     const std::function<int(const void* const*, void* const*, int64_t, cudaStream_t)>& fn,
                     int64_t min_chunk = 1) {
    int dev;
    int rc = ensure_device(&dev);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(g_host_mu[dev < 0 ? 0 : (dev >= kMaxDevices ? kMaxDevices - 1 : dev)]);
    return run_rows_host(dev, n, ins, nin, outs, nout,
                         [&](int, int64_t, int64_t rows, const void* const* d_in, void* const* d_out,
                             cudaStream_t st) -> int { return fn(d_in, d_out, rows, st); },
                         min_chunk);
}

int sa_fft_forward_host(const double* h_in, int64_t n, int64_t len, double* h_re, double* h_im) {
    SA_REQUIRE(n == 0 || (h_in && h_re && h_im), "null buffer");
    if (n < 0 || len < 1) return fail(SA_ERR_INVALID_ARG, "bad batch shape");
    const int64_t bins = len / 2 + 1;
    const HostIn in{h_in, 8 * len};
    const HostOut out[2] = {{h_re, 8 * bins}, {h_im, 8 * bins}};
    return host_rows(n, &in, 1, out, 2, [&](const void* const* di, void* const* dout, int64_t rows, cudaStream_t st) {
        return sa_fft_forward((const double*)di[0], rows, len, (double*)dout[0], (double*)dout[1], st);
    });
}

int sa_fft_inverse_host(const double* h_re, const double* h_im, int64_t n, int64_t len, double* h_out) {
    SA_REQUIRE(n == 0 || (h_re && h_im && h_out), "null buffer");
    if (n < 0 || len < 1) return fail(SA_ERR_INVALID_ARG, "bad batch shape");
    const int64_t bins = len / 2 + 1;
    const HostIn in[2] = {{h_re, 8 * bins}, {h_im, 8 * bins}};
    const HostOut out{h_out, 8 * len};
    return host_rows(n, in, 2, &out, 1, [&](const void* const* di, void* const* dout, int64_t rows, cudaStream_t st) {
        return sa_fft_inverse((const double*)di[0], (const double*)di[1], rows, len, (double*)dout[0], st);
    });
}

int sa_dct_forward_host(const double* h_in, int64_t n, int64_t len, double* h_out) {
    SA_REQUIRE(n == 0 || (h_in && h_out), "null buffer");
    if (n < 0 || len < 1) return fail(SA_ERR_INVALID_ARG, "bad batch shape");
    const HostIn in{h_in, 8 * len};
    const HostOut out{h_out, 8 * len};
    return host_rows(n, &in, 1, &out, 1, [&](const void* const* di, void* const* dout, int64_t rows, cudaStream_t st) {
        return sa_dct_forward((const double*)di[0], rows, len, (double*)dout[0], st);
    });
}

int sa_dct_inverse_host(const double* h_in, int64_t n, int64_t len, double* h_out) {
    SA_REQUIRE(n == 0 || (h_in && h_out), "null buffer");
    if (n < 0 || len < 1) return fail(SA_ERR_INVALID_ARG, "bad batch shape");
    const HostIn in{h_in, 8 * len};
    const HostOut out{h_out, 8 * len};
    return host_rows(n, &in, 1, &out, 1, [&](const void* const* di, void* const* dout, int64_t rows, cudaStream_t st) {
        return sa_dct_inverse((const double*)di[0], rows, len, (double*)dout[0], st);
    });
}

int sa_dtw_batch_host(const double* h_a, const double* h_b, int64_t n_pairs, int64_t len_a, int64_t len_b,
                      double* h_dist) {
    SA_REQUIRE(n_pairs <= 0 || (h_a && h_b && h_dist), "null buffer");
    if (n_pairs < 0 || len_a < 1 || len_b < 1) return fail(SA_ERR_INVALID_ARG, "bad batch shape");
    const HostIn in[2] = {{h_a, 8 * len_a}, {h_b, 8 * len_b}};
    const HostOut out{h_dist, 8};
    return host_rows(n_pairs, in, 2, &out, 1,
                     [&](const void* const* di, void* const* dout, int64_t rows, cudaStream_t st) {
                         return sa_dtw_batch((const double*)di[0], (const double*)di[1], rows, len_a, len_b,
                                             (double*)dout[0], st);
                     },
                     std::max<int64_t>(1, (1ll << 30) / (8 * (len_a + len_b) + 8)));  // few, large launches
}

int sa_fft_forward(const double* d_in, int64_t n, int64_t len, double* d_re, double* d_im, void* stream) {
    SA_REQUIRE(n >= 0 && len >= 1, "bad batch shape");
    SA_REQUIRE(n == 0 || (d_in && d_re && d_im), "null buffer");
    int dev;
    int rc = ensure_device(&dev);
    if (rc) return rc;
    FftParams p{};
    if (!make_fft_geo(len, &p.fft, true)) return fail(SA_ERR_UNSUPPORTED, "no FFT plan for this length");
    p.x = d_in; p.reo = d_re; p.imo = d_im; p.n = n; p.L = (int32_t)len;
    rc = get_twiddles(dev, (int)len, &p.tw);
    if (!rc) rc = finish_geo(dev, &p.fft);
    if (rc) return rc;
    if (cta_fft_len(len, {d_in})) {
        int threads, grid;
        size_t smem;
        const void* kern = pick_rfft_cta_kernel(len);
        rc = cta_launch_shape(dev, kern, len, n, &threads, &smem, &grid);
        if (rc || n == 0) return rc;
        return cta_launch(kern, grid, threads, smem, (cudaStream_t)stream, p);
    }
    size_t smem;
    int lcap, grid;
    bool global;
    rc = fft_plan_smem(dev, len, &lcap, &smem, &grid, (const void*)rfft_kernel<false>, n, &global, &p.fft);
    if (rc) return rc;
    p.lcap = lcap;
    if (n == 0) return SA_OK;
    rc = alloc_row_bufs(global, lcap, grid, (cudaStream_t)stream, &p.gbuf);
    if (rc) return rc;
    if (global) rfft_kernel<true><<<grid, 32, smem, (cudaStream_t)stream>>>(p);
    else rfft_kernel<false><<<grid, 32, smem, (cudaStream_t)stream>>>(p);
    SA_CUDA(cudaGetLastError());
    __atomic_add_fetch(&g_launches, 1, __ATOMIC_RELAXED);
    if (p.gbuf) SA_CUDA(cudaFreeAsync(p.gbuf, (cudaStream_t)stream));
    return SA_OK;
}

int sa_fft_inverse(const double* d_re, const double* d_im, int64_t n, int64_t len, double* d_out, void* stream) {
    SA_REQUIRE(n >= 0 && len >= 1, "bad batch shape");
    SA_REQUIRE(n == 0 || (d_re && d_im && d_out), "null buffer");
    int dev;
    int rc = ensure_device(&dev);
    if (rc) return rc;
    FftParams p{};
    if (!make_fft_geo(len, &p.fft, true)) return fail(SA_ERR_UNSUPPORTED, "no FFT plan for this length");
    p.re = d_re; p.im = d_im; p.xo = d_out; p.n = n; p.L = (int32_t)len;
    rc = get_twiddles(dev, (int)len, &p.tw);
    if (!rc) rc = finish_geo(dev, &p.fft);
    if (rc) return rc;
    if (cta_fft_len(len, {d_out})) {
        int threads, grid;
        size_t smem;
        const void* kern = pick_irfft_cta_kernel(len);
        rc = cta_launch_shape(dev, kern, len, n, &threads, &smem, &grid);
        if (rc || n == 0) return rc;
        return cta_launch(kern, grid, threads, smem, (cudaStream_t)stream, p);
    }
    size_t smem;
    int lcap, grid;
    bool global;
    rc = fft_plan_smem(dev, len, &lcap, &smem, &grid, (const void*)irfft_kernel<false>, n, &global, &p.fft);
    if (rc) return rc;
    p.lcap = lcap;
    if (n == 0) return SA_OK;
    rc = alloc_row_bufs(global, lcap, grid, (cudaStream_t)stream, &p.gbuf);
    if (rc) return rc;
    if (global) irfft_kernel<true><<<grid, 32, smem, (cudaStream_t)stream>>>(p);
    else irfft_kernel<false><<<grid, 32, smem, (cudaStream_t)stream>>>(p);
    SA_CUDA(cudaGetLastError());
    __atomic_add_fetch(&g_launches, 1, __ATOMIC_RELAXED);
    if (p.gbuf) SA_CUDA(cudaFreeAsync(p.gbuf, (cudaStream_t)stream));
    return SA_OK;
}

static int dct_launch(const double* d_in, int64_t n, int64_t len, double* d_out, void* stream, int inverse) {
    SA_REQUIRE(n >= 0 && len >= 1, "bad batch shape");
    SA_REQUIRE(n == 0 || (d_in && d_out), "null buffer");
    int dev;
    int rc = ensure_device(&dev);
    if (rc) return rc;
    FftParams p{};
    if (len < 1 || !make_fft_geo(len, &p.fft, true)) return fail(SA_ERR_UNSUPPORTED, "no DCT plan for this length");
    p.x = d_in; p.xo = d_out; p.n = n; p.L = (int32_t)len; p.inverse = inverse;
    rc = get_twiddles(dev, (int)len, &p.tw);
    if (rc) return rc;
    rc = get_dct_twiddles(dev, (int)len, &p.dtw);
    if (!rc) rc = finish_geo(dev, &p.fft);
    if (rc) return rc;
    if (cta_fft_len(len, {d_in, d_out})) {
        int threads, grid;
        size_t smem;
        const void* kern = inverse ? pick_dct3_cta_kernel(len) : pick_dct2_cta_kernel(len);
        rc = cta_launch_shape(dev, kern, len, n, &threads, &smem, &grid);
        if (rc || n == 0) return rc;
        return cta_launch(kern, grid, threads, smem, (cudaStream_t)stream, p);
    }
    size_t smem;
    int lcap, grid;
    bool global;
    rc = fft_plan_smem(dev, len, &lcap, &smem, &grid, (const void*)dct_kernel<false>, n, &global, &p.fft);
    if (rc) return rc;
    p.lcap = lcap;
    if (n == 0) return SA_OK;
    rc = alloc_row_bufs(global, lcap, grid, (cudaStream_t)stream, &p.gbuf);
    if (rc) return rc;
    if (global) dct_kernel<true><<<grid, 32, smem, (cudaStream_t)stream>>>(p);
    else dct_kernel<false><<<grid, 32, smem, (cudaStream_t)stream>>>(p);
    SA_CUDA(cudaGetLastError());
    __atomic_add_fetch(&g_launches, 1, __ATOMIC_RELAXED);
    if (p.gbuf) SA_CUDA(cudaFreeAsync(p.gbuf, (cudaStream_t)stream));
    return SA_OK;
}

int sa_dct_forward(const double* d_in, int64_t n, int64_t len, double* d_out, void* stream) {
    return dct_launch(d_in, n, len, d_out, stream, 0);
}

int sa_dct_inverse(const double* d_in, int64_t n, int64_t len, double* d_out, void* stream) {
    return dct_launch(d_in, n, len, d_out, stream, 1);
}

int sa_dtw_batch(const double* d_a, const double* d_b, int64_t n_pairs, int64_t len_a, int64_t len_b,
                 double* d_dist, void* stream) {
    SA_REQUIRE(n_pairs >= 0 && len_a >= 1 && len_b >= 1, "bad batch shape");
    SA_REQUIRE(n_pairs == 0 || (d_a && d_b && d_dist), "null buffer");
    int dev;
    int rc = ensure_device(&dev);
    if (rc) return rc;
    if (len_a < 1 || len_b < 1) return fail(SA_ERR_INVALID_ARG, "DTW needs non-empty series");
    DeviceState& ds = dev_state(dev);
    size_t smem = sizeof(double) * (size_t)len_b;
    const bool global = smem > ds.smem_optin;  // long b: the row buffer lives in global memory
    if (global) smem = 0;
    DtwParams p{};
    p.a = d_a; p.b = d_b; p.dist = d_dist; p.pairs = n_pairs; p.n = (int32_t)len_a; p.m = (int32_t)len_b;
    p.stage_b = 0;  // b from L1: staging it halves the resident warps (measured slower)
    if (n_pairs == 0) return SA_OK;
    int per_sm = 0;
    SA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dtw_batch_kernel<false>, 32, smem));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)ds.sms * std::max(per_sm, 1), n_pairs));
    if (global) SA_CUDA(sa_malloc_async((void**)&p.gprow, sizeof(double) * (size_t)len_b * grid, (cudaStream_t)stream));
    if (global) dtw_batch_kernel<true><<<grid, 32, smem, (cudaStream_t)stream>>>(p);
    else dtw_batch_kernel<false><<<grid, 32, smem, (cudaStream_t)stream>>>(p);
    SA_CUDA(cudaGetLastError());
    __atomic_add_fetch(&g_launches, 1, __ATOMIC_RELAXED);
    if (p.gprow) SA_CUDA(cudaFreeAsync(p.gprow, (cudaStream_t)stream));
    return SA_OK;
}

int sa_dtw_path(const double* d_a, int64_t len_a, const double* d_b, int64_t len_b, double* d_acc, int32_t* d_path,
                int32_t* d_path_len, double* d_dist, void* stream) {
    SA_REQUIRE(len_a >= 1 && len_b >= 1, "DTW needs non-empty series");
    SA_REQUIRE(d_a && d_b && d_acc && d_path && d_path_len && d_dist, "null buffer");
    int dev;
    int rc = ensure_device(&dev);
    if (rc) return rc;
    if (len_a < 1 || len_b < 1) return fail(SA_ERR_INVALID_ARG, "DTW needs non-empty series");
    DeviceState& ds = dev_state(dev);
    size_t smem = sizeof(double) * (size_t)len_b;
    const bool global = smem > ds.smem_optin;
    if (global) smem = 0;
    DtwParams p{};
    p.a = d_a; p.b = d_b; p.dist = d_dist; p.acc = d_acc;
    p.path = d_path; p.path_len = d_path_len;
    p.stage_b = 0;
    p.pairs = 1; p.n = (int32_t)len_a; p.m = (int32_t)len_b;
    if (global) SA_CUDA(sa_malloc_async((void**)&p.gprow, sizeof(double) * (size_t)len_b, (cudaStream_t)stream));
    if (global) dtw_path_kernel<true><<<1, 32, smem, (cudaStream_t)stream>>>(p);
    else dtw_path_kernel<false><<<1, 32, smem, (cudaStream_t)stream>>>(p);
    SA_CUDA(cudaGetLastError());
    __atomic_add_fetch(&g_launches, 1, __ATOMIC_RELAXED);
    if (p.gprow) SA_CUDA(cudaFreeAsync(p.gprow, (cudaStream_t)stream));
    return SA_OK;
}

int sa_repr_values(const double* d_values, int64_t n, char* d_out, int32_t* d_len, void* stream) {
    SA_REQUIRE(n >= 0 && (n == 0 || (d_values && d_out && d_len)), "bad arguments");
    int dev;
    int rc = ensure_device(&dev);
    if (rc) return rc;
    if (n == 0) return SA_OK;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)dev_state(dev).sms * 16);
    repr_values_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(d_values, n, d_out, d_len);
    SA_CUDA(cudaGetLastError());
    __atomic_add_fetch(&g_launches, 1, __ATOMIC_RELAXED);
    return SA_OK;
}

int sa_parse_values(const char* d_text, const int64_t* d_offsets, int64_t n, double* d_out, int32_t* d_ok,
                    char* d_scratch, void* stream) {
    SA_REQUIRE(n >= 0 && (n == 0 || (d_text && d_offsets && d_out && d_ok)), "bad arguments");
    int dev;
    int rc = ensure_device(&dev);
    if (rc) return rc;
    if (n == 0) return SA_OK;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)dev_state(dev).sms * 16);
    parse_values_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(d_text, d_offsets, n, d_out, d_ok, d_scratch);
    SA_CUDA(cudaGetLastError());
    __atomic_add_fetch(&g_launches, 1, __ATOMIC_RELAXED);
    return SA_OK;
}

int sa_augment_spectrum(const sa_stage* stage, uint64_t master_seed, int64_t series_offset, const double* d_re,
                        const double* d_im, int64_t n, int64_t len, double* d_re_out, double* d_im_out,
                        void* stream) {
    SA_REQUIRE(stage, "null stage");
    SA_REQUIRE(n >= 0 && len >= 1, "bad batch shape");
    SA_REQUIRE(n == 0 || (d_re && d_im && d_re_out && d_im_out), "null buffer");
    int dev;
    int rc = ensure_device(&dev);
    if (rc) return rc;
    if (!is_spectral(stage->op)) return fail(SA_ERR_INVALID_ARG, "not a spectral stage");
    SpecParams p{};
    p.st.op = stage->op;
    p.st.index = stage->index;
    p.st.prob = stage->probability;
    for (int k = 0; k < 4; ++k) {
        p.st.f[k] = stage->f[k];
        p.st.i[k] = stage->i[k];
    }
    p.seed = master_seed;
    p.offset = series_offset;
    p.re = d_re; p.im = d_im; p.reo = d_re_out; p.imo = d_im_out; p.n = n; p.L = (int32_t)len;
    size_t smem;
    int lcap, grid;
    bool global;
    rc = fft_plan_smem(dev, len, &lcap, &smem, &grid, (const void*)spectrum_kernel<false>, n, &global);
    if (rc) return rc;
    p.lcap = lcap;
    if (n == 0) return SA_OK;
    rc = alloc_row_bufs(global, lcap, grid, (cudaStream_t)stream, &p.gbuf);
    if (rc) return rc;
    if (global) spectrum_kernel<true><<<grid, 32, smem, (cudaStream_t)stream>>>(p);
    else spectrum_kernel<false><<<grid, 32, smem, (cudaStream_t)stream>>>(p);
    SA_CUDA(cudaGetLastError());
    __atomic_add_fetch(&g_launches, 1, __ATOMIC_RELAXED);
    if (p.gbuf) SA_CUDA(cudaFreeAsync(p.gbuf, (cudaStream_t)stream));
    SA_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    return SA_OK;
}

int sa_host_copy(void* dst, const void* src, int64_t bytes) {
    if (bytes < 0 || (bytes > 0 && (!dst || !src))) return fail(SA_ERR_INVALID_ARG, "sa_host_copy: bad arguments");
    CopyPool::get().copy(dst, src, (size_t)bytes);
    return SA_OK;
}

int sa_host_all_finite(const double* p, int64_t n, int32_t* all_finite) {
    if (n < 0 || !all_finite || (n > 0 && !p)) return fail(SA_ERR_INVALID_ARG, "sa_host_all_finite: bad arguments");
    // 256 KB blocks over the host cores; a block stops at its first bad word
    // (exponent all ones: NaN or +-Inf), and later blocks see the flag
    const int64_t kBlock = 1 << 15;
    const int64_t blocks = (n + kBlock - 1) / kBlock;
    std::atomic<int> bad{0};
    const uint64_t* w = reinterpret_cast<const uint64_t*>(p);
    auto scan = [&](size_t blk) {
        if (bad.load(std::memory_order_relaxed)) return;
        const int64_t lo = (int64_t)blk * kBlock, hi = std::min(n, lo + kBlock);
        uint64_t acc = 0;
        for (int64_t i = lo; i < hi; ++i) acc |= (uint64_t)((w[i] & 0x7ff0000000000000ull) == 0x7ff0000000000000ull);
        if (acc) bad.store(1, std::memory_order_relaxed);
    };
    if (blocks <= 4) {
        for (int64_t b = 0; b < blocks; ++b) scan((size_t)b);
    } else {
        // group blocks into ~4 jobs per thread so job overhead stays small
        CopyPool& pool = CopyPool::get();
        const int64_t jobs = std::min<int64_t>(blocks, 4 * (int64_t)pool.threads());
        const int64_t per = (blocks + jobs - 1) / jobs;
        pool.parallel((size_t)jobs, [&](size_t j) {
            for (int64_t b = (int64_t)j * per; b < std::min(blocks, ((int64_t)j + 1) * per); ++b) scan((size_t)b);
        });
    }
    *all_finite = bad.load() ? 0 : 1;
    return SA_OK;
}

int sa_host_alloc(void** ptr, int64_t bytes) {
    SA_REQUIRE(ptr && bytes >= 0, "bad arguments");
    SA_CUDA(cudaHostAlloc(ptr, (size_t)bytes, cudaHostAllocPortable));
    return SA_OK;
}

int sa_host_free(void* ptr) {
    SA_CUDA(cudaFreeHost(ptr));
    return SA_OK;
}

}  // extern "C"

#include "sa_dataset_host.inc"
