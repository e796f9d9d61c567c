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
// (row-major n x m) for the path backtrack.  `prow` is smem of >= m doubles.
__device__ double dtw_warp(const double* __restrict__ a, int n, const double* __restrict__ b, int m,
                           double* prow, double* acc, int lane) {
    double result = 0.0;
    for (int i0 = 0; i0 < n; i0 += 32) {
        const int i = i0 + lane;
        const double ai = i < n ? a[i] : 0.0;
        double left = 0.0, up = 0.0, diag = 0.0;
        const int steps = m + 31;
        for (int t = 0; t < steps; ++t) {
            const int j = t - lane;
            if (lane == 0 && i0 > 0 && j < m) {
                up = prow[j];
                diag = j > 0 ? prow[j - 1] : 0.0;
            }
            double v = 0.0;
            const bool live = (j >= 0) && (j < m) && (i < n);
            if (live) {
                const double c = fabs(ai - b[j]);
                if (i == 0) {
                    v = (j == 0) ? c : left + c;
                } else if (j == 0) {
                    v = up + c;
                } else {
                    double best = diag;
                    if (up < best) best = up;
                    if (left < best) best = left;
                    v = c + best;
                }
                left = v;
                if (acc) acc[(int64_t)i * m + j] = v;
                if (i == n - 1 && j == m - 1) result = v;
            }
            // lane l+1 needs this cell as its "up" next step; its diagonal is
            // the "up" it used this step
            const double nu = __shfl_up_sync(0xffffffffu, v, 1);
            __syncwarp();
            if (lane == 31 && live) prow[j] = v;
            if (lane > 0) {
                diag = up;
                up = nu;
            }
            __syncwarp();
        }
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
