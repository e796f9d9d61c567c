// rng_probe.cu -- TEST INFRASTRUCTURE ONLY (tests/test_gpu_rng_probe.py).
//
// Builds the product's warp normals() walk (paper_2601_03159_b200/csrc/
// sa_rng.cuh) with the window's word source replaced by a caller-supplied
// word array, so crafted streams can drive the ziggurat paths numpy's
// generator makes rare (runs of wedge words across lanes, a wedge head on the
// window's last word, tails, all-slow lanes) and the results can be compared
// with the C oracle's sequential random_standard_normal on the same words.
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstring>

// the "key" carries the word array: k0 = device pointer, k1 = word count
#define SA_WINDOW_BLOCK(k0, k1, b, o0, o1, o2, o3)                                  \
    do {                                                                            \
        const uint64_t* W_ = reinterpret_cast<const uint64_t*>(k0);                 \
        const uint64_t q_ = 4 * (uint64_t)(b);                                      \
        o0 = q_ + 0 < (k1) ? W_[q_ + 0] : 0x200ull;                                 \
        o1 = q_ + 1 < (k1) ? W_[q_ + 1] : 0x200ull;                                 \
        o2 = q_ + 2 < (k1) ? W_[q_ + 2] : 0x200ull;                                 \
        o3 = q_ + 3 < (k1) ? W_[q_ + 3] : 0x200ull;                                 \
    } while (0)
#include "../../paper_2601_03159_b200/csrc/sa_rng.cuh"

using namespace sa;

// One warp walks `ncalls` consecutive normals() calls of counts[c] normals on
// the stream words[0..nwords); pos[c] = stream position after call c.
// start_mode 1 starts like the chain kernel after its gate pre-pass: block 0
// cached (wn = 4) and word 0 consumed by the gate.
__global__ void probe_normals_kernel(const uint64_t* words, int64_t nwords, const int* counts, int ncalls,
                                     int start_mode, double* out, int64_t* pos) {
    __shared__ __align__(16) uint64_t winbuf[SA_WIN];
    __shared__ __align__(16) uint64_t cached[4];
    __shared__ ZigEntry zs[256];
    const int lane = threadIdx.x;
    for (int i = lane; i < 256; i += 32) zs[i] = g_zig[i];
    if (lane < 4) cached[lane] = lane < nwords ? words[lane] : 0x200ull;
    __syncwarp();
    WStream s;
    s.k0 = reinterpret_cast<uint64_t>(words);
    s.k1 = (uint64_t)nwords;
    s.has32 = 0;
    s.u32 = 0;
    s.winbuf = winbuf;
    if (start_mode == 1) {
        s.win = cached; s.wb = 0; s.wn = 4; s.wpos = 1;
    } else {
        s.win = winbuf; s.wb = 0; s.wn = 0; s.wpos = 0;
    }
    int64_t base = 0;
    for (int c = 0; c < ncalls; ++c) {
        double* o = out + base;
        normals(s, lane, counts[c], zs, [&](int k, double z) { o[k] = z; });
        if (lane == 0) pos[c] = (int64_t)s.wpos;
        base += counts[c];
    }
}

extern "C" int rngprobe_normals(const uint64_t* h_words, int64_t nwords, const int* h_counts, int ncalls,
                                int start_mode, double* h_out, int64_t* h_pos) {
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
    if (cudaMemcpyToSymbol(g_zig, zig, sizeof(zig)) != cudaSuccess) return -1;
    if (cudaMemcpyToSymbol(g_fi, fid, sizeof(fid)) != cudaSuccess) return -1;
    int64_t total = 0;
    for (int c = 0; c < ncalls; ++c) total += h_counts[c];
    uint64_t* dw = nullptr; int* dc = nullptr; double* dout = nullptr; int64_t* dpos = nullptr;
    int rc = -2;
    if (cudaMalloc(&dw, 8 * (nwords + 1)) == cudaSuccess && cudaMalloc(&dc, 4 * ncalls) == cudaSuccess &&
        cudaMalloc(&dout, 8 * (total + 1)) == cudaSuccess && cudaMalloc(&dpos, 8 * ncalls) == cudaSuccess &&
        cudaMemcpy(dw, h_words, 8 * nwords, cudaMemcpyHostToDevice) == cudaSuccess &&
        cudaMemcpy(dc, h_counts, 4 * ncalls, cudaMemcpyHostToDevice) == cudaSuccess) {
        probe_normals_kernel<<<1, 32>>>(dw, nwords, dc, ncalls, start_mode, dout, dpos);
        if (cudaDeviceSynchronize() == cudaSuccess &&
            cudaMemcpy(h_out, dout, 8 * total, cudaMemcpyDeviceToHost) == cudaSuccess &&
            cudaMemcpy(h_pos, dpos, 8 * ncalls, cudaMemcpyDeviceToHost) == cudaSuccess)
            rc = 0;
    }
    cudaFree(dw); cudaFree(dc); cudaFree(dout); cudaFree(dpos);
    return rc;
}

// sa_log1p (the restatement of the reference libm's log1p) evaluated on the
// device, for tests/test_log1p_pin.py.
__global__ void probe_log1p_kernel(const double* x, double* y, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = sa_log1p(x[i]);
}

extern "C" int rngprobe_log1p(const double* h_x, double* h_y, int64_t n) {
    double *dx = nullptr, *dy = nullptr;
    int rc = -2;
    if (cudaMalloc(&dx, 8 * (n + 1)) == cudaSuccess && cudaMalloc(&dy, 8 * (n + 1)) == cudaSuccess &&
        cudaMemcpy(dx, h_x, 8 * n, cudaMemcpyHostToDevice) == cudaSuccess) {
        probe_log1p_kernel<<<592, 256>>>(dx, dy, n);
        if (cudaDeviceSynchronize() == cudaSuccess && cudaMemcpy(h_y, dy, 8 * n, cudaMemcpyDeviceToHost) == cudaSuccess)
            rc = 0;
    }
    cudaFree(dx); cudaFree(dy);
    return rc;
}
