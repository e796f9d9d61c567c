// FP64 FMA peak of one B200 (the compute-side roofline denominator for the
// FFT-bearing configs): 16 independent DFMA chains per
// thread, full occupancy.  Prints JSON: {"fp64_fma_tflops": ..., ...}.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) fma_kernel(int iters, double x, double y, double* out) {
    double a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = fma(a[i], x, y);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    double* out;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    fma_kernel<<<blocks, threads>>>(iters, 0.999999, 1e-7, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        fma_kernel<<<blocks, threads>>>(iters, 0.999999, 1e-7, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    const double fmas = (double)blocks * threads * iters * 16;
    const double tflops = 2.0 * fmas / (best / 1e3) / 1e12;
    printf("{\"fp64_fma_tflops\": %.3f, \"fma_per_clk_per_sm\": %.1f, \"sms\": %d, \"max_clock_mhz\": %d, "
           "\"kernel_ms\": %.4f, \"method\": \"16 independent DFMA chains per thread, %d x %d threads, best of 5\"}\n",
           tflops, fmas / (best / 1e3) / sms / (clk * 1e3), sms, clk / 1000, best, blocks, threads);
    return cudaGetLastError() != cudaSuccess;
}
