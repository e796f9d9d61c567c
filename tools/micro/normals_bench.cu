// Micro-benchmark of the warp ziggurat walk (sa_rng.cuh normals()) with a
// jitter-style emit (x[k] += sigma z in shared memory), 12 warps per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2601_03159_b200/csrc/sa_rng.cuh"

using namespace sa;

template <int MODE, int NT>
__global__ void __launch_bounds__(NT, 1) bench(int rows_per_warp, int L, double* out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    ZigEntry* zs = reinterpret_cast<ZigEntry*>(smem);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) zs[i] = g_zig[i];
    double* x = reinterpret_cast<double*>(smem + 4096) + w * (L + 128 + 8);
    uint64_t* win = reinterpret_cast<uint64_t*>(x + L + 8);
    for (int t = lane; t < L; t += 32) x[t] = t;
    __syncthreads();
    double acc = 0;
    for (int q = 0; q < rows_per_warp; ++q) {
        uint64_t k0, k1;
        derive_key(5, 0, (uint64_t)(blockIdx.x * (NT / 32) + w) * rows_per_warp + q, k0, k1);
        WStream s;
        s.k0 = k0; s.k1 = k1; s.winbuf = win; s.win = win; s.wb = 0; s.wn = 0; s.wpos = 1; s.has32 = 0; s.u32 = 0;
        if (MODE == 0) {
            normals(s, lane, L, zs, [&](int k, double z) { x[k] = x[k] + (0.0 + 0.05 * z); });
        } else {
            normals(s, lane, L, zs, [&](int k, double z) { acc += z * (double)k; });
        }
        __syncwarp();
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + x[lane];
}

template <int MODE, int NT>
void run(const char* name, double* out, int sms, int L) {
    const int rpw = 64 * 12 / (NT / 32);
    const size_t sm = 4096 + (NT / 32) * (L + 136) * 8;
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, bench<MODE, NT>);
    printf("regs %d local %zu  ", fa.numRegs, fa.localSizeBytes);
    cudaFuncSetAttribute(bench<MODE, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    bench<MODE, NT><<<sms, NT, sm>>>(rpw, L, out);
    cudaEventRecord(a);
    for (int k = 0; k < 5; ++k) bench<MODE, NT><<<sms, NT, sm>>>(rpw, L, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double rows = 5.0 * sms * (NT / 32) * rpw;
    printf("%-44s %8.3f ms  %.1f SM-cycles per warp-row of %d normals  (err %s)\n", name, ms / 5,
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
    double* out;
    cudaMalloc(&out, sms * 1024 * 8);
    run<0, 384>("jitter emit, 12 warps", out, sms, 1024);
    run<0, 512>("jitter emit, 16 warps", out, sms, 1024);
    run<0, 640>("jitter emit, 20 warps", out, sms, 1024);
    run<0, 768>("jitter emit, 24 warps", out, sms, 1024);
    run<0, 1024>("jitter emit, 32 warps", out, sms, 1024);
    return 0;
}
