// dist.cu -- data-plane kernels of the sharded multi-GPU step (sm_100a).
//
// The reference's worker exchanges (engine.py:201-237, 499-507;
// distributed.py:127-226) re-designed for one process per GPU with
// Gaussian-wise shards and pixel ROW BANDS (contiguous tile rows per GPU):
//
//   route   : per visible shard row, the contiguous range of bands its tile
//             rect overlaps; (band, row) pairs are emitted in row order and
//             stably grouped by band, then packed into 80-byte records
//             (depth key, global id, rect, 12 raster features) for one
//             all-to-all.  Rows stay in ascending global id inside every
//             band group, so the receiver's concatenation (source order) is
//             already id-ascending and the stable depth sort reproduces the
//             single-GPU (depth, id) order exactly.
//   blocks  : the renderer folds each splat's (tile, splat) subtotals per
//             canonical block of `canon` tile rows (tiles ascending inside a
//             block, float64) and emits one record per (splat, block) for the
//             splat's owner.  Bands are unions of whole blocks, so the owner's
//             fold of block sums in (band, block) order is bit-identical to
//             the single-GPU two-level fold -- the run is bitwise independent
//             of the GPU count, the reference's headline property.
//   fold    : the owner groups received records by shard row (stable) and
//             sums them in arrival order (bands ascending).
#include <type_traits>

#include "common.cuh"
#include "radix.cuh"

namespace isg {

constexpr int MAX_BANDS = 64;

struct Bands {
    int n;
    int start[MAX_BANDS + 1];  // tile-row boundaries, start[n] = tiles_y
};

__device__ __forceinline__ int band_of(const Bands &b, int row) {
    int lo = 0, hi = b.n - 1;  // last band with start <= row
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (b.start[mid] <= row) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// ------------------------------------------------------------ routing --
// A visible splat reaches the contiguous band range [lo, hi] its tile rect's
// rows overlap.  Per band it carries three weights: 1 splat record, nb
// canonical-block gradient records (blocks of `canon` tile rows inside the
// band) and its tile entries in the band (the band's list length).
__device__ __forceinline__ void splat_bands(const Bands &b, const int4 rc, int &lo, int &hi) {
    lo = band_of(b, rc.y);
    hi = band_of(b, rc.w);
}

struct BandWeights {
    int64_t nb, tiles;
};

__device__ __forceinline__ BandWeights band_weights(const Bands &b, const int4 rc, int d,
                                                    int canon) {
    const int y0 = max(rc.y, b.start[d]), y1 = min(rc.w, b.start[d + 1] - 1);
    BandWeights w;
    w.nb = (int64_t)(y1 / canon - y0 / canon + 1);
    w.tiles = (int64_t)(rc.z - rc.x + 1) * (int64_t)(y1 - y0 + 1);
    return w;
}

constexpr int PLAN_T = 256;  // shard rows per plan block (route_plan/pack, owner_fold)

// Per plan block and band: (splat records, block records) in plan[blk][d][0..1]
// and the tile entries in tiles_blk[blk][d].  Bands are visited over the
// block's band range with warp reductions (no contended shared atomics).
__global__ void __launch_bounds__(PLAN_T) route_plan_kernel(int64_t n,
                                                            const uint8_t *__restrict__ flag,
                                                            const int4 *__restrict__ rect,
                                                            Bands bands, int canon,
                                                            int64_t *__restrict__ plan,
                                                            int64_t *__restrict__ tiles_blk) {
    __shared__ long long s_w[3][PLAN_T / 32];
    __shared__ int s_lo, s_hi;
    const int nbands = bands.n;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i = (int64_t)blockIdx.x * PLAN_T + threadIdx.x;
    int lo = nbands, hi = -1;
    int4 rc = make_int4(0, 0, -1, -1);
    if (i < n && flag[i]) {
        rc = rect[i];
        splat_bands(bands, rc, lo, hi);
    }
    if (threadIdx.x == 0) {
        s_lo = nbands;
        s_hi = -1;
    }
    __syncthreads();
    if (hi >= lo) {
        atomicMin(&s_lo, lo);
        atomicMax(&s_hi, hi);
    }
    __syncthreads();
    const int blo = s_lo, bhi = s_hi;
    int64_t *pb = plan + 2 * (int64_t)blockIdx.x * nbands;
    int64_t *tb = tiles_blk + (int64_t)blockIdx.x * nbands;
    for (int d = threadIdx.x; d < nbands; d += PLAN_T) {
        if (d < blo || d > bhi) {
            pb[2 * d] = pb[2 * d + 1] = 0;
            tb[d] = 0;
        }
    }
    for (int d = blo; d <= bhi; d++) {
        long long c = 0, nb = 0, t = 0;
        if (lo <= d && d <= hi) {
            const BandWeights w = band_weights(bands, rc, d, canon);
            c = 1;
            nb = w.nb;
            t = w.tiles;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            c += __shfl_xor_sync(0xffffffffu, c, o);
            nb += __shfl_xor_sync(0xffffffffu, nb, o);
            t += __shfl_xor_sync(0xffffffffu, t, o);
        }
        if (lane == 0) {
            s_w[0][warp] = c;
            s_w[1][warp] = nb;
            s_w[2][warp] = t;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            long long a0 = 0, a1 = 0, a2 = 0;
#pragma unroll
            for (int w = 0; w < PLAN_T / 32; w++) {
                a0 += s_w[0][w];
                a1 += s_w[1][w];
                a2 += s_w[2][w];
            }
            pb[2 * d] = a0;
            pb[2 * d + 1] = a1;
            tb[d] = a2;
        }
        __syncthreads();
    }
}

// One CTA per band: exclusive prefix over the plan blocks of the two record
// counts (in place) and the band totals (records, block records, tiles).
__global__ void __launch_bounds__(1024) route_scan_kernel(int64_t nblk, int nbands,
                                                          int64_t *__restrict__ plan,
                                                          const int64_t *__restrict__ tiles_blk,
                                                          int64_t *__restrict__ totals) {
    __shared__ long long sw0[32], sw1[32], s_tiles[32];
    const int d = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    long long carry0 = 0, carry1 = 0, tiles = 0;
    for (int64_t c = 0; c < nblk; c += 1024) {
        const int64_t b = c + threadIdx.x;
        int64_t *p = plan + 2 * (b * nbands + d);
        const long long v0 = b < nblk ? p[0] : 0, v1 = b < nblk ? p[1] : 0;
        tiles += b < nblk ? tiles_blk[b * nbands + d] : 0;
        long long x0 = v0, x1 = v1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y0 = __shfl_up_sync(0xffffffffu, x0, o);
            const long long y1 = __shfl_up_sync(0xffffffffu, x1, o);
            if (lane >= o) {
                x0 += y0;
                x1 += y1;
            }
        }
        if (lane == 31) {
            sw0[warp] = x0;
            sw1[warp] = x1;
        }
        __syncthreads();
        long long b0 = carry0, b1 = carry1, t0 = 0, t1 = 0;
        for (int w = 0; w < 32; w++) {
            if (w < warp) {
                b0 += sw0[w];
                b1 += sw1[w];
            }
            t0 += sw0[w];
            t1 += sw1[w];
        }
        if (b < nblk) {
            p[0] = b0 + x0 - v0;
            p[1] = b1 + x1 - v1;
        }
        carry0 += t0;
        carry1 += t1;
        __syncthreads();
    }
    for (int o = 16; o > 0; o >>= 1) tiles += __shfl_xor_sync(0xffffffffu, tiles, o);
    if (lane == 0) s_tiles[warp] = tiles;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int w = 0; w < 32; w++) t += s_tiles[w];
        totals[3 * d] = carry0;
        totals[3 * d + 1] = carry1;
        totals[3 * d + 2] = t;
    }
}

// In-block exclusive prefix of `v` over the CTA's threads (thread order =
// shard row order); `total` is the CTA total.  All threads must call.
template <int T>
__device__ __forceinline__ int64_t block_excl(int64_t v, int64_t *s_warp, int64_t &total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    int64_t before = 0;
    total = 0;
#pragma unroll
    for (int w = 0; w < T / 32; w++) {
        const int64_t t = s_warp[w];
        if (w < warp) before += t;
        total += t;
    }
    __syncthreads();
    return before + x - v;
}

// Where band d's segment of this shard's records starts: a local send or
// receive buffer, or -- the peer-store exchange -- band d's receive buffers
// on its own GPU, mapped into this process (NVLink loads/stores).
struct PackDest {
    uint64_t *keys[MAX_BANDS];
    int4 *pay[MAX_BANDS];  // 4 int4 per record
};

// Splat records of every visible shard row for each band it reaches, in
// shard row order inside each band's segment: the depth key (8 B) and a
// 64-byte payload (rect, 12 raster features), stored straight to the
// segment's destination (own band: this rank's receive buffers; peer
// exchange: the band's receive buffers on its GPU).
__global__ void __launch_bounds__(PLAN_T) route_pack_kernel(
    int64_t n, const uint8_t *__restrict__ flag, const int4 *__restrict__ rect,
    const uint64_t *__restrict__ key, const int4 *__restrict__ feat, Bands bands,
    const int64_t *__restrict__ plan, PackDest dst) {
    __shared__ int64_t s_warp[PLAN_T / 32];
    __shared__ int s_lo, s_hi;
    const int nbands = bands.n;
    const int64_t i = (int64_t)blockIdx.x * PLAN_T + threadIdx.x;
    int lo = nbands, hi = -1;
    int4 rc = make_int4(0, 0, -1, -1);
    if (i < n && flag[i]) {
        rc = rect[i];
        splat_bands(bands, rc, lo, hi);
    }
    if (threadIdx.x == 0) {
        s_lo = nbands;
        s_hi = -1;
    }
    __syncthreads();
    if (hi >= lo) {
        atomicMin(&s_lo, lo);
        atomicMax(&s_hi, hi);
    }
    __syncthreads();
    const int blo = s_lo, bhi = s_hi;
    const int64_t *pb = plan + 2 * (int64_t)blockIdx.x * nbands;
    for (int d = blo; d <= bhi; d++) {
        const bool on = lo <= d && d <= hi;
        int64_t tot;
        const int64_t ex = block_excl<PLAN_T>(on ? 1 : 0, s_warp, tot);
        if (on) {
            const int64_t slot = pb[2 * d] + ex;
            int4 *pp = dst.pay[d] + 4 * slot;
            dst.keys[d][slot] = key[i];
            pp[0] = rc;
            pp[1] = feat[3 * i];
            pp[2] = feat[3 * i + 1];
            pp[3] = feat[3 * i + 2];
        }
    }
}

// The reference's round-robin routing (_route_mask, _kernels.py:378-394):
// row i reaches worker w iff its tile rect touches a tile whose linear id is
// congruent to w modulo the worker count.
__global__ void route_mask_kernel(int64_t n, const int4 *__restrict__ rects, int tiles_x,
                                  int workers, uint8_t *__restrict__ mask) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int4 rc = rects[i];
    const uint64_t full = workers == 64 ? ~0ull : (1ull << workers) - 1ull;
    uint64_t seen = 0;
    for (int ty = rc.y; ty <= rc.w && seen != full; ty++)
        for (int tx = rc.x; tx <= rc.z && seen != full; tx++)
            seen |= 1ull << (((int64_t)ty * tiles_x + tx) % workers);
    for (int w = 0; w < workers; w++) mask[i * workers + w] = (uint8_t)((seen >> w) & 1ull);
}

// Canonical blocks of each received splat inside the band.
__global__ void band_blocks_kernel(int64_t r, const int4 *__restrict__ pay, int row_lo,
                                   int row_hi, int canon, int64_t *__restrict__ nb) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= r) return;
    const int4 rc = pay[4 * k];
    const int y0 = max(rc.y, row_lo), y1 = min(rc.w, row_hi - 1);
    nb[k] = y1 >= y0 ? (int64_t)(y1 / canon - y0 / canon + 1) : 0;
}
// ------------------------------------------------------ gradient fold --
// Band side: every rank's (tile, splat) subtotals are folded per canonical
// block (tiles ascending inside the block, float64) and each block sum is
// written as a 9-double record at gpos[order[r]] + b: records are laid out by
// RECEIVE index, so the segment that goes back to source rank s is exactly
// its splats in its shard row order.  Streaming as in reduce_ordered_f32:
// every warp owns 32 consecutive ranks whose slots are one contiguous span,
// staged through shared memory with TMA bulk copies (cp.async.bulk +
// mbarrier, double buffered).
constexpr int BF_WARPS = 4;
constexpr int BF_THREADS = 32 * BF_WARPS;
constexpr int BF_SLOTS = 96;

__device__ __forceinline__ void bf_mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar)),
                 "r"(count)
                 : "memory");
}
__device__ __forceinline__ void bf_bulk_load(void *dst, const void *src, unsigned bytes,
                                             uint64_t *bar) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"((unsigned)__cvta_generic_to_shared(dst)),
        "l"(src), "r"(bytes), "r"(b)
        : "memory");
}
__device__ __forceinline__ void bf_mbar_wait(uint64_t *bar, unsigned parity) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(b), "r"(parity)
            : "memory");
    }
}

// One rank's block sums, emitted as they close (same arithmetic as FoldState).
struct BlockEmit {
    double bs[9];
    int y, w, dx, canon;
    bool open;
    double *out;

    __device__ __forceinline__ void init(int4 rc, int row_lo, int canon_rows, double *o) {
        y = max(rc.y, row_lo);
        w = rc.z - rc.x + 1;
        dx = 0;
        canon = canon_rows;
        open = false;
        out = o;
#pragma unroll
        for (int k = 0; k < 9; k++) bs[k] = 0.0;
    }
    __device__ __forceinline__ void close() {
#pragma unroll
        for (int k = 0; k < 9; k++) {
            out[k] = bs[k];
            bs[k] = 0.0;
        }
        out += 9;
        open = false;
    }
    __device__ __forceinline__ void step(const float *v) {
#pragma unroll
        for (int k = 0; k < 9; k++) bs[k] += (double)v[k];
        open = true;
        if (++dx == w) {
            dx = 0;
            y++;
            if (y % canon == 0) close();
        }
    }
    __device__ __forceinline__ void finish() {
        if (open) close();
    }
};

// Live-only layout: rows from the records (float 9), a record for every block
// of the rank's clipped rows in the band (zero when no slot of it is live).
struct BlockEmitLive {
    double bs[9];
    int blk, last, canon;
    double *out;

    __device__ __forceinline__ void init(int4 rc, int row_lo, int row_hi, int canon_rows,
                                         double *o) {
        canon = canon_rows;
        blk = max(rc.y, row_lo) / canon;
        last = min(rc.w, row_hi - 1) / canon;
        out = o;
#pragma unroll
        for (int k = 0; k < 9; k++) bs[k] = 0.0;
    }
    __device__ __forceinline__ void close() {
#pragma unroll
        for (int k = 0; k < 9; k++) {
            out[k] = bs[k];
            bs[k] = 0.0;
        }
        out += 9;
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

// Destination of the gradient records by source rank: receive indices
// [recv_end[s-1], recv_end[s]) came from source s, whose records go to
// base[s] + 9 * gpos (a local buffer, or -- the peer-store exchange -- the
// owner's receive buffer on its GPU, base offset so gpos lands in place).
struct GradDest {
    double *base[MAX_BANDS];
    int64_t recv_end[MAX_BANDS];
};

template <bool LIVE>
__global__ void __launch_bounds__(BF_THREADS) band_fold_kernel(
    int64_t m, const int64_t *__restrict__ emit_off, const float *__restrict__ partials,
    const int4 *__restrict__ rect_sorted, const int32_t *__restrict__ order,
    const int64_t *__restrict__ gpos, int row_lo, int row_hi, int canon, GradDest dst) {
    constexpr int PS = partial_stride<float>();
    __shared__ __align__(128) float sbuf[BF_WARPS][2][BF_SLOTS * PS];
    __shared__ __align__(8) uint64_t sbar[BF_WARPS][2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r0 = ((int64_t)blockIdx.x * BF_WARPS + warp) * 32;
    if (r0 >= m) return;
    const int64_t r = r0 + lane;
    const bool live = r < m;
    const int64_t span0 = emit_off[r0];
    const int64_t span1 = emit_off[min(r0 + 32, m)];
    int64_t p = live ? emit_off[r] : 0;
    const int64_t p1 = live ? emit_off[r + 1] : 0;
    double *out = dst.base[0];
    if (live) {
        const int32_t q = order[r];
        int src = 0;
        while (q >= dst.recv_end[src]) src++;
        out = dst.base[src] + 9 * gpos[q];
    }
    typename std::conditional<LIVE, BlockEmitLive, BlockEmit>::type st;
    if constexpr (LIVE) {
        st.init(live ? rect_sorted[r] : make_int4(0, 0, -1, -1), row_lo, row_hi, canon, out);
    } else {
        st.init(live ? rect_sorted[r] : make_int4(0, 0, 0, 0), row_lo, canon, out);
    }
    const int nch = (int)((span1 - span0 + BF_SLOTS - 1) / BF_SLOTS);
    float(*buf)[BF_SLOTS * PS] = sbuf[warp];
    uint64_t *bar = sbar[warp];
    auto issue = [&](int k) {
        const int64_t c0 = span0 + (int64_t)k * BF_SLOTS;
        const unsigned cnt = (unsigned)min((int64_t)BF_SLOTS, span1 - c0);
        bf_bulk_load(buf[k & 1], partials + PS * c0, cnt * PS * (unsigned)sizeof(float),
                     &bar[k & 1]);
    };
    if (lane == 0) {
        bf_mbar_init(&bar[0], 1);
        bf_mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (nch > 0) issue(0);
        if (nch > 1) issue(1);
    }
    __syncwarp();
    for (int k = 0; k < nch; k++) {
        bf_mbar_wait(&bar[k & 1], (unsigned)((k >> 1) & 1));
        const int64_t c0 = span0 + (int64_t)k * BF_SLOTS;
        const int64_t e = min(p1, c0 + BF_SLOTS);
        const float *b = buf[k & 1];
        for (; p < e; p++) st.step(b + PS * (p - c0));
        __syncwarp();
        if (lane == 0 && k + 2 < nch) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(k + 2);
        }
    }
    if (live) st.finish();
}

// Raster cost of the band per canonical block: sum over its pixels of n_last
// (the backward's last list position, a proxy of both raster passes), added
// as integers to a float64 histogram over all blocks of the image (exact:
// integer sums below 2^53 do not depend on the order of the atomics).
__global__ void __launch_bounds__(256) band_cost_kernel(const int32_t *__restrict__ n_last,
                                                        int prow0, int width, int block_px_rows,
                                                        double *__restrict__ hist) {
    const int row = blockIdx.x;  // pixel row inside the band
    const int32_t *p = n_last + (int64_t)row * width;
    long long s = 0;
    for (int x = threadIdx.x; x < width; x += 256) s += p[x];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __shared__ long long sw[8];
    if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int w = 0; w < 8; w++) t += sw[w];
        atomicAdd(hist + (prow0 + row) / block_px_rows, (double)t);
    }
}

struct SegPtrs {
    const double *seg[MAX_BANDS];  // band d's gradient records for this shard
};

// Owner side (reduce_gradients_fused, distributed.py:178-226): per shard row,
// its block records from every band it reached, bands ascending then blocks
// ascending -- the canonical two-level order -- summed in float64.  Record
// positions come from the route plan (the same per-band prefix the band used
// to lay them out), so nothing is sorted.  Rows not visible get zeros.
__global__ void __launch_bounds__(PLAN_T) owner_fold_plan_kernel(
    int64_t n, const uint8_t *__restrict__ flag, const int4 *__restrict__ rect, Bands bands,
    int canon, const int64_t *__restrict__ plan, SegPtrs segs, double *__restrict__ grad2d) {
    __shared__ int64_t s_warp[PLAN_T / 32];
    __shared__ int s_lo, s_hi;
    const int nbands = bands.n;
    const int64_t i = (int64_t)blockIdx.x * PLAN_T + threadIdx.x;
    int lo = nbands, hi = -1;
    int4 rc = make_int4(0, 0, -1, -1);
    if (i < n && flag[i]) {
        rc = rect[i];
        splat_bands(bands, rc, lo, hi);
    }
    if (threadIdx.x == 0) {
        s_lo = nbands;
        s_hi = -1;
    }
    __syncthreads();
    if (hi >= lo) {
        atomicMin(&s_lo, lo);
        atomicMax(&s_hi, hi);
    }
    __syncthreads();
    const int blo = s_lo, bhi = s_hi;
    const int64_t *pb = plan + 2 * (int64_t)blockIdx.x * nbands;
    double acc[9];
#pragma unroll
    for (int k = 0; k < 9; k++) acc[k] = 0.0;
    for (int d = blo; d <= bhi; d++) {
        const bool on = lo <= d && d <= hi;
        const int64_t nb = on ? band_weights(bands, rc, d, canon).nb : 0;
        int64_t tot;
        const int64_t ex = block_excl<PLAN_T>(nb, s_warp, tot);
        const double *src = segs.seg[d] + 9 * (pb[2 * d + 1] + ex);
        for (int64_t b = 0; b < nb; b++) {
#pragma unroll
            for (int k = 0; k < 9; k++) acc[k] += src[9 * b + k];
        }
    }
    if (i < n) {
#pragma unroll
        for (int k = 0; k < 9; k++) grad2d[9 * i + k] = acc[k];
    }
}
__global__ void grad_rows_kernel(int64_t r, const int32_t *__restrict__ rec, uint32_t *__restrict__ rows,
                                 int32_t *__restrict__ idx) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= r) return;
    rows[k] = (uint32_t)rec[20 * k];
    idx[k] = (int32_t)k;
}

// Owner fold: rows sorted (stable) -> per row the records in arrival order.
__global__ void owner_fold_kernel(int64_t n_rows, const int32_t *__restrict__ seg_off,
                                  const int32_t *__restrict__ perm, const int32_t *__restrict__ rec,
                                  double *__restrict__ grad2d) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_rows) return;
    const int a = seg_off[i], b = seg_off[i + 1];
    if (a == b) return;  // not visible: the chain rule never reads this row
    double acc[9];
#pragma unroll
    for (int q = 0; q < 9; q++) acc[q] = 0.0;
    for (int k = a; k < b; k++) {
        const double *d = reinterpret_cast<const double *>(rec + 20 * (int64_t)perm[k] + 2);
#pragma unroll
        for (int q = 0; q < 9; q++) acc[q] += d[q];
    }
#pragma unroll
    for (int q = 0; q < 9; q++) grad2d[9 * i + q] = acc[q];
}


inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace isg

using namespace isg;

// Exclusive scan of n int64 counts into off[0..n] (off[0] = 0) and *total.
extern "C" int isg_scan_i64(void *workspace, size_t *ws_bytes, int64_t n, const int64_t *cnt,
                            int64_t *off, int64_t *total, void *stream) {
    if (!ws_bytes || n < 0 || n > INT32_MAX) return (int)cudaErrorInvalidValue;
    const size_t need = scan_i64_ws_bytes(n);
    if (!workspace) {
        *ws_bytes = need;
        return 0;
    }
    if (*ws_bytes < need) return (int)cudaErrorInvalidValue;
    return scan_i64(workspace, *ws_bytes, n, cnt, off, total, (cudaStream_t)stream);
}

static int fill_bands(Bands &b, const int32_t *band_rows, int32_t n_bands) {
    if (n_bands < 1 || n_bands > MAX_BANDS || !band_rows) return 1;
    b.n = n_bands;
    for (int i = 0; i <= n_bands; i++) b.start[i] = band_rows[i];
    return 0;
}

extern "C" int isg_route_plan_size(int64_t n, int32_t n_bands, int64_t *plan_elems) {
    if (n < 0 || n_bands < 1 || n_bands > MAX_BANDS || !plan_elems)
        return (int)cudaErrorInvalidValue;
    const int64_t nblk = (n + PLAN_T - 1) / PLAN_T;
    *plan_elems = 3 * nblk * n_bands;  // plan (2 per band) + tiles (1 per band)
    return 0;
}

extern "C" int isg_route_plan(int64_t n, const uint8_t *flag, const int32_t *rect,
                              const int32_t *band_rows, int32_t n_bands, int32_t canon_rows,
                              int64_t *plan, int64_t *totals, void *stream) {
    Bands b;
    if (n < 0 || canon_rows < 1 || fill_bands(b, band_rows, n_bands) || !plan || !totals)
        return (int)cudaErrorInvalidValue;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nblk = (n + PLAN_T - 1) / PLAN_T;
    if (nblk == 0) {
        cudaError_t e = cudaMemsetAsync(totals, 0, sizeof(int64_t) * 3 * n_bands, s);
        return (int)e;
    }
    int64_t *tiles_blk = plan + 2 * nblk * n_bands;
    route_plan_kernel<<<(unsigned)nblk, PLAN_T, 0, s>>>(n, flag, (const int4 *)rect, b,
                                                        canon_rows, plan, tiles_blk);
    ISG_CHECK_LAUNCH();
    route_scan_kernel<<<n_bands, 1024, 0, s>>>(nblk, n_bands, plan, tiles_blk, totals);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_route_pack(int64_t n, const uint8_t *flag, const int32_t *rect,
                              const uint64_t *key, const float *feat, const int32_t *band_rows,
                              int32_t n_bands, const int64_t *plan, const int64_t *dest_off,
                              int32_t self_band, uint64_t *keys_send, int32_t *pay_send,
                              uint64_t *keys_self, int32_t *pay_self, void *stream) {
    Bands b;
    if (n < 0 || fill_bands(b, band_rows, n_bands) || !dest_off || self_band < -1 ||
        self_band >= n_bands)
        return (int)cudaErrorInvalidValue;
    const int64_t nblk = (n + PLAN_T - 1) / PLAN_T;
    if (nblk == 0) return 0;
    PackDest dst;
    for (int d = 0; d < n_bands; d++) {
        const bool self = d == self_band;
        dst.keys[d] = (self ? keys_self : keys_send) + dest_off[d];
        dst.pay[d] = (int4 *)(self ? pay_self : pay_send) + 4 * dest_off[d];
    }
    route_pack_kernel<<<(unsigned)nblk, PLAN_T, 0, (cudaStream_t)stream>>>(
        n, flag, (const int4 *)rect, key, (const int4 *)feat, b, plan, dst);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_route_pack_peer(int64_t n, const uint8_t *flag, const int32_t *rect,
                                   const uint64_t *key, const float *feat,
                                   const int32_t *band_rows, int32_t n_bands, const int64_t *plan,
                                   uint64_t *const *keys_dst, int32_t *const *pay_dst,
                                   void *stream) {
    Bands b;
    if (n < 0 || fill_bands(b, band_rows, n_bands) || !keys_dst || !pay_dst)
        return (int)cudaErrorInvalidValue;
    const int64_t nblk = (n + PLAN_T - 1) / PLAN_T;
    if (nblk == 0) return 0;
    PackDest dst;
    for (int d = 0; d < n_bands; d++) {
        dst.keys[d] = keys_dst[d];
        dst.pay[d] = (int4 *)pay_dst[d];
        if ((reinterpret_cast<uintptr_t>(pay_dst[d]) & 15) != 0) return (int)cudaErrorInvalidValue;
    }
    route_pack_kernel<<<(unsigned)nblk, PLAN_T, 0, (cudaStream_t)stream>>>(
        n, flag, (const int4 *)rect, key, (const int4 *)feat, b, plan, dst);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_route_mask(int64_t n, const int32_t *rects, int32_t tiles_x, int32_t workers,
                              uint8_t *mask, void *stream) {
    if (n < 0 || tiles_x <= 0 || workers < 1 || workers > 64 || (n > 0 && (!rects || !mask)))
        return (int)cudaErrorInvalidValue;
    if (n == 0) return 0;
    route_mask_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
        n, (const int4 *)rects, tiles_x, workers, mask);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_band_blocks(int64_t r, const int32_t *payload, int32_t row_lo, int32_t row_hi,
                               int32_t canon_rows, int64_t *nb, void *stream) {
    if (r < 0 || canon_rows < 1) return (int)cudaErrorInvalidValue;
    if (r == 0) return 0;
    band_blocks_kernel<<<blocks_for(r, 256), 256, 0, (cudaStream_t)stream>>>(
        r, (const int4 *)payload, row_lo, row_hi, canon_rows, nb);
    ISG_CHECK_LAUNCH();
    return 0;
}

static int launch_band_fold(int64_t m, const int64_t *emit_off, const float *partials,
                            const int32_t *rect_sorted, const int32_t *order, const int64_t *gpos,
                            int row_lo, int row_hi, int canon, int live_layout,
                            const GradDest &dst, cudaStream_t s) {
    if (live_layout)
        band_fold_kernel<true><<<blocks_for(m, BF_THREADS), BF_THREADS, 0, s>>>(
            m, emit_off, partials, (const int4 *)rect_sorted, order, gpos, row_lo, row_hi, canon,
            dst);
    else
        band_fold_kernel<false><<<blocks_for(m, BF_THREADS), BF_THREADS, 0, s>>>(
            m, emit_off, partials, (const int4 *)rect_sorted, order, gpos, row_lo, row_hi, canon,
            dst);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_band_fold(int64_t m, const int64_t *emit_off, const float *partials,
                             const int32_t *rect_sorted, const int32_t *order,
                             const int64_t *gpos, int32_t row_lo, int32_t row_hi,
                             int32_t canon_rows, int32_t live_layout, double *gbuf, void *stream) {
    if (m < 0 || canon_rows < 1) return (int)cudaErrorInvalidValue;
    if (m == 0) return 0;
    GradDest dst;
    dst.base[0] = gbuf;
    dst.recv_end[0] = INT64_MAX;
    return launch_band_fold(m, emit_off, partials, rect_sorted, order, gpos, row_lo, row_hi,
                            canon_rows, live_layout, dst, (cudaStream_t)stream);
}

extern "C" int isg_band_fold_peer(int64_t m, const int64_t *emit_off, const float *partials,
                                  const int32_t *rect_sorted, const int32_t *order,
                                  const int64_t *gpos, int32_t row_lo, int32_t row_hi,
                                  int32_t canon_rows, int32_t live_layout, int32_t n_src,
                                  const int64_t *recv_end, double *const *dst_base,
                                  void *stream) {
    if (m < 0 || canon_rows < 1 || n_src < 1 || n_src > MAX_BANDS || !recv_end || !dst_base)
        return (int)cudaErrorInvalidValue;
    if (m == 0) return 0;
    if (recv_end[n_src - 1] < m) return (int)cudaErrorInvalidValue;
    GradDest dst;
    for (int s = 0; s < n_src; s++) {
        dst.base[s] = dst_base[s];
        dst.recv_end[s] = recv_end[s];
    }
    for (int s = n_src; s < MAX_BANDS; s++) dst.recv_end[s] = INT64_MAX;
    return launch_band_fold(m, emit_off, partials, rect_sorted, order, gpos, row_lo, row_hi,
                            canon_rows, live_layout, dst, (cudaStream_t)stream);
}

extern "C" int isg_band_cost(const int32_t *n_last, int32_t prow0, int32_t prow1, int32_t width,
                              int32_t canon_rows, double *hist, void *stream) {
    if (prow0 < 0 || prow1 < prow0 || width <= 0 || canon_rows < 1)
        return (int)cudaErrorInvalidValue;
    if (prow1 == prow0) return 0;
    band_cost_kernel<<<prow1 - prow0, 256, 0, (cudaStream_t)stream>>>(n_last, prow0, width,
                                                                     16 * canon_rows, hist);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_owner_fold_plan(int64_t n, const uint8_t *flag, const int32_t *rect,
                                   const int32_t *band_rows, int32_t n_bands, int32_t canon_rows,
                                   const int64_t *plan, const double *const *seg,
                                   double *grad2d, void *stream) {
    Bands b;
    if (n < 0 || canon_rows < 1 || fill_bands(b, band_rows, n_bands) || !seg)
        return (int)cudaErrorInvalidValue;
    const int64_t nblk = (n + PLAN_T - 1) / PLAN_T;
    if (nblk == 0) return 0;
    SegPtrs sp;
    for (int d = 0; d < n_bands; d++) sp.seg[d] = seg[d];
    owner_fold_plan_kernel<<<(unsigned)nblk, PLAN_T, 0, (cudaStream_t)stream>>>(
        n, flag, (const int4 *)rect, b, canon_rows, plan, sp, grad2d);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_grad_rows(int64_t r, const int32_t *records, uint32_t *rows, int32_t *idx,
                             void *stream) {
    if (r < 0) return (int)cudaErrorInvalidValue;
    if (r == 0) return 0;
    grad_rows_kernel<<<blocks_for(r, 256), 256, 0, (cudaStream_t)stream>>>(r, records, rows, idx);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_owner_fold(int64_t n_rows, const int32_t *seg_off, const int32_t *perm,
                              const int32_t *records, double *grad2d, void *stream) {
    if (n_rows < 0) return (int)cudaErrorInvalidValue;
    if (n_rows == 0) return 0;
    owner_fold_kernel<<<blocks_for(n_rows, 256), 256, 0, (cudaStream_t)stream>>>(
        n_rows, seg_off, perm, records, grad2d);
    ISG_CHECK_LAUNCH();
    return 0;
}

// Device-to-device copy on the stream; either side may be a peer GPU's
// memory mapped into this process (the halo rows of the peer exchange).
extern "C" int isg_copy(void *dst, const void *src, int64_t bytes, void *stream) {
    if (bytes < 0 || (bytes > 0 && (!dst || !src))) return (int)cudaErrorInvalidValue;
    if (bytes == 0) return 0;
    return (int)cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice,
                                (cudaStream_t)stream);
}
