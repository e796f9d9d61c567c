// Throughput of the 52/53-bit integer -> double conversions of the ziggurat
// and random() paths: I2F.F64.U64 against the exponent-splice form
// as_double(0x433.. | v) - 2^52 (one LOP3 + one DADD), and the sign flip as
// DADD + FSEL against an XOR of the sign bit.  Prints SMSP cycles per warp
// instruction group at 3 warps per SMSP (the chain kernel's occupancy).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(384) conv_kernel(int iters, uint64_t seed, double* out, long long* cyc) {
    uint64_t v[8];
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        v[i] = (seed * (threadIdx.x + 1 + 977 * i)) & 0x000fffffffffffffULL;
        acc[i] = 0.0;
    }
    const long long t0 = clock64();
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            double d;
            if (MODE == 0) {
                d = (double)v[i];
            } else {
                d = __longlong_as_double((long long)(v[i] | 0x4330000000000000ULL)) - 4503599627370496.0;
            }
            acc[i] += d;
            v[i] = (v[i] + 0x9E3779B97F4AULL) & 0x000fffffffffffffULL;
        }
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
static double run(int sms) {
    const int iters = 4096;
    double* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(double) * sms * 384);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    conv_kernel<MODE><<<sms, 384>>>(iters, 0x2545F4914F6CDD1DULL, out, cyc);
    conv_kernel<MODE><<<sms, 384>>>(iters, 0x2545F4914F6CDD1DULL, out, cyc);
    cudaDeviceSynchronize();
    long long h[256];
    cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += (double)h[i];
    avg /= sms;
    cudaFree(out);
    cudaFree(cyc);
    // 3 warps per SMSP, 8 conversions per iteration each
    return avg / (iters * 8.0 * 3.0);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double a = run<0>(sms), b = run<1>(sms);
    printf("{\"i2f_f64_u64_smsp_cycles_per_warp_group\": %.2f, \"splice_dadd_smsp_cycles_per_warp_group\": %.2f, "
           "\"note\": \"group = conversion + DADD accumulate + 64-bit add/and; 12 warps per SM\"}\n", a, b);
    return cudaGetLastError() != cudaSuccess;
}
