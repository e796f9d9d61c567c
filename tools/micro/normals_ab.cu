// A/B of the ziggurat walks in sa_rng.cuh: normals (strided rows) vs
// normals_blocked (4 consecutive words per lane): identical draws and stream
// positions on many streams (count per stream varied), then timing.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>
#include "../../paper_2601_03159_b200/csrc/sa_rng.cuh"

using namespace sa;

__global__ void __launch_bounds__(384) check(int rows_per_warp, unsigned long long* mism, unsigned long long* total) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    ZigEntry* zs = reinterpret_cast<ZigEntry*>(smem);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) zs[i] = g_zig[i];
    double* a = reinterpret_cast<double*>(smem + 4096) + w * (2 * 1100 + 2 * 128 + 8);
    double* b = a + 1100;
    uint64_t* win1 = reinterpret_cast<uint64_t*>(b + 1100);
    uint64_t* win2 = win1 + 128;
    __syncthreads();
    unsigned long long bad = 0, cnt = 0;
    for (int q = 0; q < rows_per_warp; ++q) {
        const uint64_t row = (uint64_t)(blockIdx.x * 12 + w) * rows_per_warp + q;
        uint64_t k0, k1;
        derive_key(7, row & 7, row, k0, k1);
        // cached block 0 (the gate pre-pass) as the chain kernel sets it up
        uint64_t c[4];
        philox(k0, k1, 1, c[0], c[1], c[2], c[3]);
        WStream s1, s2;
        s1.k0 = s2.k0 = k0; s1.k1 = s2.k1 = k1;
        s1.win = s2.win = c; s1.winbuf = win1; s2.winbuf = win2;
        s1.wb = s2.wb = 0; s1.wn = s2.wn = 4; s1.wpos = s2.wpos = 1; s1.has32 = s2.has32 = 0; s1.u32 = s2.u32 = 0;
        // several calls with varying counts (stream continues across calls)
        for (int call = 0; call < 3; ++call) {
            const int count = call == 0 ? 1 + (int)(row % 1024) : (call == 1 ? 1 + (int)((row * 7) % 300) : 1026);
            for (int t = lane; t < count; t += 32) { a[t] = -1.0; b[t] = -2.0; }
            __syncwarp();
            normals(s1, lane, count, zs, [&](int kk, double z) { a[kk] = z; });
            normals_blocked(s2, lane, count, zs, [&](int kk, double z) { b[kk] = z; });
            __syncwarp();
            for (int t = lane; t < count; t += 32) {
                uint64_t x, y;
                memcpy(&x, &a[t], 8);
                memcpy(&y, &b[t], 8);
                bad += x != y;
            }
            if (lane == 0) { bad += (s1.wpos != s2.wpos); cnt += count; }
            __syncwarp();
        }
    }
    atomicAdd(mism, bad);
    atomicAdd(total, cnt);
}

template <int MODE>
__global__ void __launch_bounds__(384) bench(int rows_per_warp, int L, double* out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    ZigEntry* zs = reinterpret_cast<ZigEntry*>(smem);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) zs[i] = g_zig[i];
    double* x = reinterpret_cast<double*>(smem + 4096) + w * (L + 128 + 8);
    uint64_t* win = reinterpret_cast<uint64_t*>(x + L + 8);
    for (int t = lane; t < L; t += 32) x[t] = t;
    __syncthreads();
    for (int q = 0; q < rows_per_warp; ++q) {
        uint64_t k0, k1;
        derive_key(5, 0, (uint64_t)(blockIdx.x * 12 + w) * rows_per_warp + q, k0, k1);
        WStream s;
        s.k0 = k0; s.k1 = k1; s.winbuf = win; s.win = win; s.wb = 0; s.wn = 0; s.wpos = 1; s.has32 = 0; s.u32 = 0;
        if (MODE == 0) normals(s, lane, L, zs, [&](int k, double z) { x[k] = x[k] + (0.0 + 0.05 * z); });
        else normals_blocked(s, lane, L, zs, [&](int k, double z) { x[k] = x[k] + (0.0 + 0.05 * z); });
        __syncwarp();
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x[lane];
}

template <int MODE>
void run(const char* name, double* out, int sms, int L) {
    const int rpw = 64;
    const size_t sm = 4096 + 12 * (L + 136) * 8;
    cudaFuncSetAttribute(bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    bench<MODE><<<sms, 384, sm>>>(rpw, L, out);
    cudaEventRecord(a);
    for (int k = 0; k < 5; ++k) bench<MODE><<<sms, 384, sm>>>(rpw, L, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double rows = 5.0 * sms * 12 * rpw;
    printf("%-36s %8.3f ms  %.1f SM-cycles per warp-row of %d normals (%s)\n", name, ms / 5,
           (ms / 1e3) * 1.965e9 * sms / rows, L, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    static const uint64_t ki[256] = SA_ZIG_KI_DOUBLE_INIT;
    static const uint64_t wi[256] = SA_ZIG_WI_DOUBLE_INIT;
    static const uint64_t fi[256] = SA_ZIG_FI_DOUBLE_INIT;
    ZigEntry z[256];
    for (int i = 0; i < 256; ++i) { z[i].ki = ki[i]; memcpy(&z[i].wi, &wi[i], 8); }
    cudaMemcpyToSymbol(g_zig, z, sizeof(z));
    cudaMemcpyToSymbol(g_fi, fi, sizeof(fi));
    unsigned long long *d, h[2];
    cudaMalloc(&d, 16);
    cudaMemset(d, 0, 16);
    const size_t smc = 4096 + 12 * (2 * 1100 + 2 * 128 + 8) * 8;
    cudaFuncSetAttribute(check, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smc);
    check<<<sms, 384, smc>>>(200, d, d + 1);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("check: %llu mismatches over %llu normals (%s)\n", h[0], h[1], cudaGetErrorString(cudaGetLastError()));
    double* out;
    cudaMalloc(&out, sms * 384 * 8);
    run<0>("strided normals (new)", out, sms, 1024);
    run<1>("blocked normals (old)", out, sms, 1024);
    run<0>("strided normals (new)", out, sms, 1024);
    run<1>("blocked normals (old)", out, sms, 1024);
    return 0;
}
