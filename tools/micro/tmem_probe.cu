// TMEM staging probe: alloc, tcgen05.st 32x32b.x8, wait, tcgen05.ld, dealloc.
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tmem_probe tools/micro/tmem_probe.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int VAR>
__global__ void probe(uint32_t* out, int cols_per_warp) {
    __shared__ uint32_t s_tmem;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    uint32_t cols = 32;
    while (cols < (uint32_t)(((nw + 3) / 4) * cols_per_warp)) cols <<= 1;
    if (wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "r"(cols) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t ta = s_tmem + ((uint32_t)(32 * (wid & 3)) << 16) + (uint32_t)((wid >> 2) * cols_per_warp);
    uint32_t v[8];
    for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * 100 + i + blockIdx.x * 100000;
    if (VAR == 1) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(ta),
                     "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        uint32_t r[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(ta) : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint32_t ok = 1;
        for (int i = 0; i < 8; ++i) ok &= (r[i] == v[i]);
        out[blockIdx.x * blockDim.x + threadIdx.x] = ok;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (wid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(cols) : "memory");
    }
}
int main() {
    uint32_t* d; cudaMalloc(&d, 4 << 20);
    int cfg[][3] = {{1, 32, 32}, {4, 32, 1}, {4, 24, 1}, {12, 104, 148}, {16, 104, 148}, {3, 24, 300}};
    for (auto& c : cfg) {
        cudaMemset(d, 0, 4 << 20);
        probe<1><<<c[2], 32 * c[0]>>>(d, c[1]);
        cudaError_t e = cudaDeviceSynchronize();
        int n = c[2] * 32 * c[0];
        uint32_t* h = new uint32_t[n];
        cudaMemcpy(h, d, 4 * n, cudaMemcpyDeviceToHost);
        int good = 0; for (int i = 0; i < n; ++i) good += h[i];
        printf("warps=%d cols=%d grid=%d: %s, %d/%d ok\n", c[0], c[1], c[2], cudaGetErrorString(e), good, n);
        delete[] h;
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
