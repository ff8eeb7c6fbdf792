// fold.cuh -- the canonical per-splat fold of (tile, splat) gradient subtotals.
//
// _reduce_scratch (_kernels.py:398-411) sums a splat's subtotals in ascending
// tile order.  Here the sum is two-level and fixed: float64 block sums over
// `canon_rows` tile rows (tiles ascending inside a block), then block sums
// ascending -- the grouping every row band of the multi-GPU step also uses,
// so the result is bitwise independent of the GPU count (canon_rows = 0: one
// plain ascending sum).  A rank's slots are contiguous and already in
// ascending tile order (emit_off, rect_sorted from isg_bin_count).
#pragma once
#include <stdint.h>

namespace isg {

template <typename T>
__device__ __forceinline__ void fold_rank(const T *__restrict__ partials, int64_t p0, int64_t p1,
                                          const int4 *__restrict__ rect_sorted, int64_t r,
                                          int row_lo, int canon_rows, double (&acc)[9]) {
    int y0 = 0, w = 1;
    if (canon_rows > 0 && p1 > p0) {
        const int4 rc = rect_sorted[r];
        y0 = max(rc.y, row_lo);
        w = rc.z - rc.x + 1;
    }
    double bs[9];
#pragma unroll
    for (int k = 0; k < 9; k++) acc[k] = bs[k] = 0.0;
    int cur = -1, dy = 0, dx = 0;
    for (int64_t p = p0; p < p1; p++) {
        const int blk = canon_rows > 0 ? (y0 + dy) / canon_rows : 0;
        if (blk != cur) {
#pragma unroll
            for (int k = 0; k < 9; k++) {
                acc[k] += bs[k];
                bs[k] = 0.0;
            }
            cur = blk;
        }
        const T *v = partials + 9 * p;
#pragma unroll
        for (int k = 0; k < 9; k++) bs[k] += (double)__ldg(v + k);
        if (++dx == w) {
            dx = 0;
            dy++;
        }
    }
#pragma unroll
    for (int k = 0; k < 9; k++) acc[k] += bs[k];
}

}  // namespace isg
