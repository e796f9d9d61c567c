// Micro-benchmark of Philox4x64-10 block throughput on one B200 (variants of
// the 64x64->128 multiply and of where the key schedule lives).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o philox_bench philox_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void mul_a(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
    lo = a * b;
    hi = __umul64hi(a, b);
}
// explicit 32-bit partial products with carry-chained mad.wide / madc
__device__ __forceinline__ void mul_b(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
    uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32), b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
    uint32_t r0, r1, r2, r3;
    asm("{\n\t"
        "mul.lo.u32 %0, %4, %6;\n\t"
        "mul.hi.u32 %1, %4, %6;\n\t"
        "mad.lo.cc.u32 %1, %4, %7, %1;\n\t"
        "madc.hi.u32 %2, %4, %7, 0;\n\t"
        "mad.lo.cc.u32 %1, %5, %6, %1;\n\t"
        "madc.hi.cc.u32 %2, %5, %6, %2;\n\t"
        "madc.hi.u32 %3, %5, %7, 0;\n\t"
        "mad.lo.cc.u32 %2, %5, %7, %2;\n\t"
        "addc.u32 %3, %3, 0;\n\t"
        "}"
        : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
        : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
    lo = ((uint64_t)r1 << 32) | r0;
    hi = ((uint64_t)r3 << 32) | r2;
}
// mul.wide.u32 pieces summed in 64-bit
__device__ __forceinline__ void mul_c(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
    uint64_t a0 = (uint32_t)a, a1 = a >> 32, b0 = (uint32_t)b, b1 = b >> 32;
    uint64_t p00 = a0 * b0, p01 = a0 * b1, p10 = a1 * b0, p11 = a1 * b1;
    uint64_t mid = (p00 >> 32) + (uint32_t)p01 + (uint32_t)p10;
    lo = (mid << 32) | (uint32_t)p00;
    hi = p11 + (p01 >> 32) + (p10 >> 32) + (mid >> 32);
}

template <int V>
__device__ __forceinline__ void mulhilo(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
    if (V == 0) mul_a(a, b, hi, lo);
    else if (V == 1) mul_b(a, b, hi, lo);
    else mul_c(a, b, hi, lo);
}

template <int V>
__device__ __forceinline__ void philox(uint64_t k0, uint64_t k1, uint64_t ctr0, uint64_t& o0, uint64_t& o1,
                                       uint64_t& o2, uint64_t& o3) {
    uint64_t c0 = ctr0, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B97F4A7C15ULL;
            k1 += 0xBB67AE8584CAA73BULL;
        }
        uint64_t hi0, lo0, hi1, lo1;
        mulhilo<V>(0xD2E7470EE14C6C93ULL, c0, hi0, lo0);
        mulhilo<V>(0xCA5A826395121157ULL, c2, hi1, lo1);
        uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    o0 = c0; o1 = c1; o2 = c2; o3 = c3;
}
template <int V>
__device__ __forceinline__ void philox2(uint64_t k0, uint64_t k1, uint64_t ca, uint64_t cb, uint64_t& a0,
                                        uint64_t& a1, uint64_t& a2, uint64_t& a3, uint64_t& b0, uint64_t& b1,
                                        uint64_t& b2, uint64_t& b3) {
    uint64_t c0 = ca, c1 = 0, c2 = 0, c3 = 0, d0 = cb, d1 = 0, d2 = 0, d3 = 0;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B97F4A7C15ULL;
            k1 += 0xBB67AE8584CAA73BULL;
        }
        uint64_t hi0, lo0, hi1, lo1, hj0, lj0, hj1, lj1;
        mulhilo<V>(0xD2E7470EE14C6C93ULL, c0, hi0, lo0);
        mulhilo<V>(0xCA5A826395121157ULL, c2, hi1, lo1);
        mulhilo<V>(0xD2E7470EE14C6C93ULL, d0, hj0, lj0);
        mulhilo<V>(0xCA5A826395121157ULL, d2, hj1, lj1);
        uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        uint64_t m0 = hj1 ^ d1 ^ k0, m2 = hj0 ^ d3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        d0 = m0; d1 = lj1; d2 = m2; d3 = lj0;
    }
    a0 = c0; a1 = c1; a2 = c2; a3 = c3;
    b0 = d0; b1 = d1; b2 = d2; b3 = d3;
}
// precomputed round keys (the warp-uniform schedule as data, e.g. in smem)
template <int V>
__device__ __forceinline__ void philox_rk(const uint64_t* rk, uint64_t ctr0, uint64_t& o0, uint64_t& o1,
                                          uint64_t& o2, uint64_t& o3) {
    uint64_t c0 = ctr0, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint64_t hi0, lo0, hi1, lo1;
        mulhilo<V>(0xD2E7470EE14C6C93ULL, c0, hi0, lo0);
        mulhilo<V>(0xCA5A826395121157ULL, c2, hi1, lo1);
        uint64_t n0 = hi1 ^ c1 ^ rk[2 * r], n2 = hi0 ^ c3 ^ rk[2 * r + 1];
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    o0 = c0; o1 = c1; o2 = c2; o3 = c3;
}

// MODE 0: keys from memory (per-warp, not provably uniform); 1: keys as
// kernel parameters (uniform registers); 2: round keys from shared memory
template <int V, int MODE>
__global__ void __launch_bounds__(384) bench(const uint64_t* keys, uint64_t pk0, uint64_t pk1, int iters,
                                             uint64_t* out) {
    __shared__ uint64_t rk[12][20];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t k0 = MODE == 1 ? pk0 : keys[2 * (blockIdx.x * 12 + w)];
    uint64_t k1 = MODE == 1 ? pk1 : keys[2 * (blockIdx.x * 12 + w) + 1];
    if (MODE == 2 && lane == 0) {
        uint64_t a = k0, b = k1;
        for (int r = 0; r < 10; ++r) {
            rk[w][2 * r] = a;
            rk[w][2 * r + 1] = b;
            a += 0x9E3779B97F4A7C15ULL;
            b += 0xBB67AE8584CAA73BULL;
        }
    }
    __syncwarp();
    uint64_t acc = 0;
    if (MODE == 3) {
        for (int i = 0; i < iters; i += 2) {
            uint64_t a0, a1, a2, a3, b0, b1, b2, b3;
            const uint64_t ctr = (uint64_t)i * 32 + lane + 1;
            philox2<V>(k0, k1, ctr, ctr + 32, a0, a1, a2, a3, b0, b1, b2, b3);
            acc ^= a0 ^ a1 ^ a2 ^ a3 ^ b0 ^ b1 ^ b2 ^ b3;
        }
        out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
        return;
    }
    for (int i = 0; i < iters; ++i) {
        uint64_t o0, o1, o2, o3;
        const uint64_t ctr = (uint64_t)i * 32 + lane + 1;
        if (MODE == 2) philox_rk<V>(rk[w], ctr, o0, o1, o2, o3);
        else philox<V>(k0, k1, ctr, o0, o1, o2, o3);
        acc ^= o0 ^ o1 ^ o2 ^ o3;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int V, int MODE>
void run(const char* name, uint64_t* keys, uint64_t* out, int sms) {
    const int iters = 4096;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    bench<V, MODE><<<sms, 384>>>(keys, 1, 2, iters, out);
    cudaEventRecord(a);
    for (int k = 0; k < 5; ++k) bench<V, MODE><<<sms, 384>>>(keys, 1, 2, iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double blocks = 5.0 * sms * 384.0 * iters;
    printf("%-40s %8.3f ms  %.3f Gblocks/s  %.1f SM-cycles per warp-block (at 1.965 GHz)\n", name, ms / 5,
           blocks / (ms / 1e3) / 1e9, (ms / 1e3) * 1.965e9 * sms / (blocks / 32), 0.0);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint64_t *keys, *out;
    cudaMalloc(&keys, 2 * 12 * sms * 8);
    cudaMemset(keys, 7, 2 * 12 * sms * 8);
    cudaMalloc(&out, sms * 384 * 8);
    run<0, 0>("umul64hi, keys from memory", keys, out, sms);
    run<0, 3>("umul64hi, 2 blocks per lane interleaved", keys, out, sms);
    run<1, 0>("ptx mad.cc chain, keys from memory", keys, out, sms);
    run<2, 0>("mul.wide pieces, keys from memory", keys, out, sms);
    run<0, 1>("umul64hi, keys as params (uniform)", keys, out, sms);
    run<1, 1>("ptx mad.cc chain, keys as params", keys, out, sms);
    run<0, 2>("umul64hi, round keys in smem", keys, out, sms);
    run<1, 2>("ptx mad.cc chain, round keys in smem", keys, out, sms);
    return 0;
}
