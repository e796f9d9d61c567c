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
// (the previous strip's last row), >= 2 m with stage_b (then a copy of b).
//
// Boundary cells use +inf for missing neighbours, so every cell is
// c + min(diag, up, left) (the first cell: c + 0); min selects one of the
// already-final neighbours and the single addition is the reference's, so
// the values are bitwise dtw.py's.  Within a strip lane 31 writes column
// t - 31 of prow while lane 0 reads columns t and t - 1: no step-level
// barrier is needed, only one per strip.
__device__ double dtw_warp(const double* __restrict__ a, int n, const double* __restrict__ b, int m,
                           double* prow, double* acc, int lane, bool stage_b) {
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    const double* bs = b;
    if (stage_b) {
        double* cp = prow + m;
        for (int j = lane; j < m; j += 32) cp[j] = b[j];
        __syncwarp();
        bs = cp;
    }
    double result = 0.0;
    for (int i0 = 0; i0 < n; i0 += 32) {
        const int i = i0 + lane;
        const double ai = i < n ? a[i] : 0.0;
        // lane 0 of the first strip sits on row 0: no row above
        double left = INF, up = INF, diag = (i == 0) ? 0.0 : INF;
        const int steps = m + 31;
        for (int t = 0; t < steps; ++t) {
            const int j = t - lane;
            const bool jin = (j >= 0) && (j < m);
            const int jc = jin ? j : 0;
            if (lane == 0 && i0 > 0 && jin) {
                up = prow[jc];
                diag = j > 0 ? prow[jc - 1] : INF;
            }
            const double c = fabs(ai - bs[jc]);
            const double best = fmin(fmin(diag, up), left);
            double v = c + best;
            const bool live = jin && (i < n);
            v = live ? v : INF;
            if (live) {
                left = v;
                if (acc) acc[(int64_t)i * m + j] = v;
                if (i == n - 1 && j == m - 1) result = v;
            }
            // lane l+1 needs this cell as its "up" next step; its diagonal is
            // the "up" it used this step
            const double nu = __shfl_up_sync(0xffffffffu, v, 1);
            if (lane == 31 && live) prow[j] = v;
            if (lane > 0) {
                diag = up;
                up = nu;
            }
            if (i == 0 && j == 0) diag = INF;  // row 0 after its first cell: no row above
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
