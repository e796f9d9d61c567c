// sa_dtw.cuh -- dynamic time warping (reference dtw.py:40-106), one warp per
// (a, b) pair.
//
// acc[i][j] = |a_i - b_j| + min(acc[i-1][j-1], acc[i-1][j], acc[i][j-1]) with
// the first row / column accumulated (dtw.py:49-62).  Each cell is ONE
// addition of its cost to a min of already-final neighbours, so any
// evaluation order gives bitwise the reference's values.  The warp sweeps
// 32-row strips along anti-diagonals: lane l owns row i0 + l and at step t
// computes column t - l; the up / diagonal neighbours come from lane l-1 by
// shuffle, lane 0 reads them from the previous strip's last row kept in
// shared memory.
#pragma once
#include <stdint.h>

namespace sa {

// Returns acc[n-1][m-1]; if acc != nullptr every cell is also stored
// (row-major n x m) for the path backtrack.  `prow` is smem of >= m doubles
// (the previous strip's last row).
//
// 64-row strips, two rows per lane (i0 + l and i0 + 32 + l: two independent
// dependency chains per step).  At step t lane l computes columns t - l and
// t - 32 - l.  Up / diagonal neighbours come from lane l-1 by shuffle; the
// second half's lane 0 takes its "up" from lane 31's first half one step
// earlier (a rotating shuffle), the first half's lane 0 from the previous
// strip's last row in prow.  Boundary cells use +inf for missing
// neighbours, so every cell is c + min(diag, up, left) (the first cell:
// c + 0): min selects one of the already-final neighbours and the single
// addition is the reference's, so the values are bitwise dtw.py's.  Within a
// strip lane 31 writes column t - 63 of prow while lane 0 reads columns t and
// t - 1: one barrier per strip suffices.
__device__ double dtw_warp(const double* __restrict__ a, int n, const double* __restrict__ b, int m,
                           double* prow, double* acc, int lane, bool /*stage_b*/) {
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    double result = 0.0;
    for (int i0 = 0; i0 < n; i0 += 64) {
        const int r1 = i0 + lane, r2 = r1 + 32;
        const double a1 = r1 < n ? a[r1] : 0.0, a2 = r2 < n ? a[r2] : 0.0;
        double left1 = INF, up1 = INF, diag1 = (r1 == 0) ? 0.0 : INF;
        double left2 = INF, up2 = INF, diag2 = INF;
        const int steps = m + 63;
        // full strip, no path: the steps where every lane's two cells are in
        // range (t in [63, m)) run a branch-free body
        const bool lean = acc == nullptr && i0 + 64 <= n;
        const int t_lo = lean ? 63 : steps, t_hi = lean ? m : steps;
        for (int t = 0; t < steps; ++t) {
            if (t == t_lo && t_lo < t_hi) {
                const double* pb1 = b + (t - lane);
                const double* pb2 = pb1 - 32;
                const bool l0 = lane == 0, l31 = lane == 31, first = i0 == 0;
                for (; t < t_hi; ++t, ++pb1, ++pb2) {
                    const int j1 = t - lane;
                    if (l0 && !first) {
                        up1 = prow[j1];
                        diag1 = prow[j1 - 1];
                    }
                    const double v1 = fabs(a1 - *pb1) + fmin(fmin(diag1, up1), left1);
                    const double v2 = fabs(a2 - *pb2) + fmin(fmin(diag2, up2), left2);
                    left1 = v1;
                    left2 = v2;
                    const double nu1 = __shfl_up_sync(0xffffffffu, v1, 1);
                    const double nu2 = __shfl_sync(0xffffffffu, l31 ? v1 : v2, (lane + 31) & 31);
                    if (l31) prow[j1 - 32] = v2;
                    if (!l0) {
                        diag1 = up1;
                        up1 = nu1;
                    }
                    diag2 = up2;
                    up2 = nu2;
                }
                if (t >= steps) break;
            }
            const int j1 = t - lane, j2 = j1 - 32;
            const bool in1 = (j1 >= 0) && (j1 < m), in2 = (j2 >= 0) && (j2 < m);
            if (lane == 0 && i0 > 0 && in1) {
                up1 = prow[j1];
                diag1 = j1 > 0 ? prow[j1 - 1] : INF;
            }
            const double b1 = b[in1 ? j1 : 0], b2 = b[in2 ? j2 : 0];
            const bool live1 = in1 && (r1 < n), live2 = in2 && (r2 < n);
            double v1 = fabs(a1 - b1) + fmin(fmin(diag1, up1), left1);
            double v2 = fabs(a2 - b2) + fmin(fmin(diag2, up2), left2);
            v1 = live1 ? v1 : INF;
            v2 = live2 ? v2 : INF;
            if (live1) {
                left1 = v1;
                if (acc) acc[(int64_t)r1 * m + j1] = v1;
                if (r1 == n - 1 && j1 == m - 1) result = v1;
            }
            if (live2) {
                left2 = v2;
                if (acc) acc[(int64_t)r2 * m + j2] = v2;
                if (r2 == n - 1 && j2 == m - 1) result = v2;
            }
            // next step's "up": lane l-1's cell; lane 0's second row: lane 31's first row
            const double nu1 = __shfl_up_sync(0xffffffffu, v1, 1);
            const double nu2 = __shfl_sync(0xffffffffu, lane == 31 ? v1 : v2, (lane + 31) & 31);
            if (lane == 31 && live2) prow[j2] = v2;
            if (lane > 0) {
                diag1 = up1;
                up1 = nu1;
            }
            diag2 = up2;
            up2 = nu2;
            if (r1 == 0 && j1 == 0) diag1 = INF;  // row 0 after its first cell: no row above
        }
        __syncwarp();
    }
    // the cell (n-1, m-1) belongs to lane (n-1) % 32
    return __shfl_sync(0xffffffffu, result, (n - 1) & 31);
}

// Reference backtrack (dtw.py:64-82): ties prefer the diagonal, then (i-1, j),
// then (i, j-1).  Single thread; writes (i, j) pairs from (0,0) forward.
__device__ int dtw_backtrack(const double* acc, int n, int m, int* path) {
    int len = 0;
    int i = n - 1, j = m - 1;
    path[2 * len] = i;
    path[2 * len + 1] = j;
    ++len;
    while (i > 0 || j > 0) {
        if (i == 0) {
            j -= 1;
        } else if (j == 0) {
            i -= 1;
        } else {
            double best = acc[(int64_t)(i - 1) * m + (j - 1)];
            int si = i - 1, sj = j - 1;
            if (acc[(int64_t)(i - 1) * m + j] < best) {
                best = acc[(int64_t)(i - 1) * m + j];
                si = i - 1;
                sj = j;
            }
            if (acc[(int64_t)i * m + (j - 1)] < best) {
                si = i;
                sj = j - 1;
            }
            i = si;
            j = sj;
        }
        path[2 * len] = i;
        path[2 * len + 1] = j;
        ++len;
    }
    // reverse in place to run from (0, 0)
    for (int p = 0, q = len - 1; p < q; ++p, --q) {
        int ti = path[2 * p], tj = path[2 * p + 1];
        path[2 * p] = path[2 * q];
        path[2 * p + 1] = path[2 * q + 1];
        path[2 * q] = ti;
        path[2 * q + 1] = tj;
    }
    return len;
}

}  // namespace sa
