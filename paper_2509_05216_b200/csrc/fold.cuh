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

#include "common.cuh"

namespace isg {

// Running state of one rank's fold; step() consumes the next slot's 9 terms.
struct FoldState {
    double acc[9], bs[9];
    int y, w, dx, canon;
    bool flush;

    __device__ __forceinline__ void init(const int4 *__restrict__ rect_sorted, int64_t r,
                                         int64_t n_slots, int row_lo, int canon_rows) {
        y = 0;
        w = 1;
        if (canon_rows > 0 && n_slots > 0) {
            const int4 rc = rect_sorted[r];
            y = max(rc.y, row_lo);
            w = rc.z - rc.x + 1;
        }
        canon = canon_rows;
        dx = 0;
        flush = false;
#pragma unroll
        for (int k = 0; k < 9; k++) acc[k] = bs[k] = 0.0;
    }

    // Block sums close where a new tile row starts a new canon block (the
    // only place the block index (row / canon) can change).
    template <typename V>
    __device__ __forceinline__ void step(const V *v) {
        if (flush) {
#pragma unroll
            for (int k = 0; k < 9; k++) {
                acc[k] += bs[k];
                bs[k] = 0.0;
            }
            flush = false;
        }
#pragma unroll
        for (int k = 0; k < 9; k++) bs[k] += (double)v[k];
        if (++dx == w) {
            dx = 0;
            y++;
            flush = canon > 0 && y % canon == 0;
        }
    }

    __device__ __forceinline__ void finish() {
#pragma unroll
        for (int k = 0; k < 9; k++) acc[k] += bs[k];
    }
};

// The same fold over the live-only layout (isg_bin_emit_live): a rank's slots
// are its composited tiles only, each record carrying its tile row (int32 bits
// in float 9).  Every canonical block of the rank's clipped rows closes in
// order -- blocks without a slot add a zero block sum -- so the sequence of
// block sums, and the result, is the full-layout fold's.
struct FoldLive {
    double acc[9], bs[9];
    int blk, last, canon;

    __device__ __forceinline__ void init(const int4 *__restrict__ rect_sorted, int64_t r,
                                         int row_lo, int row_hi, int canon_rows) {
        const int4 rc = rect_sorted[r];
        canon = canon_rows;
        blk = max(rc.y, row_lo) / canon;
        last = min(rc.w, row_hi - 1) / canon;
#pragma unroll
        for (int k = 0; k < 9; k++) acc[k] = bs[k] = 0.0;
    }
    __device__ __forceinline__ void close() {
#pragma unroll
        for (int k = 0; k < 9; k++) {
            acc[k] += bs[k];
            bs[k] = 0.0;
        }
        blk++;
    }
    __device__ __forceinline__ void step(const float *v) {
        const int b = __float_as_int(v[9]) / canon;
        while (blk < b) close();
#pragma unroll
        for (int k = 0; k < 9; k++) bs[k] += (double)v[k];
    }
    __device__ __forceinline__ void finish() {
        while (blk <= last) close();
    }
};

template <typename T>
__device__ __forceinline__ void fold_rank(const T *__restrict__ partials, int64_t p0, int64_t p1,
                                          const int4 *__restrict__ rect_sorted, int64_t r,
                                          int row_lo, int canon_rows, double (&acc)[9]) {
    FoldState st;
    st.init(rect_sorted, r, p1 - p0, row_lo, canon_rows);
    for (int64_t p = p0; p < p1; p++) st.step(partials + partial_stride<T>() * p);
    st.finish();
#pragma unroll
    for (int k = 0; k < 9; k++) acc[k] = st.acc[k];
}

}  // namespace isg
