// binning.cu -- global depth order and per-tile CSR lists (sm_100a).
//
// Replaces np.lexsort((indices, depth)) (rasterizer.py:161-163,
// engine.py:213-215) and build_tile_lists (rasterizer.py:166-191 over
// _kernels.py:202-225).  The depth order is a stable LSD radix sort of the
// fp64 depth bits (positive doubles order like their bit patterns) over
// values already in ascending global-id order, so ties break on the id
// exactly like lexsort.  Tile lists are built by duplicating each rank into
// (tile, rank) pairs in rank order and stably sorting on the tile id, so each
// tile's list is in global compositing order -- bit-identical to the
// reference's count/cumsum/fill.  All kernels are HBM-bound integer work.
#include "common.cuh"
#include "radix.cuh"
#include "raster_common.cuh"

namespace isg {

#ifndef GATHER_T
#define GATHER_T 256
#endif
#ifndef EMIT_T
#define EMIT_T 256
#endif
__global__ void __launch_bounds__(GATHER_T) gather_rank_kernel(
    int64_t n, const uint64_t *__restrict__ sorted_keys, const int32_t *__restrict__ order,
    const int4 *__restrict__ rect, int rect_stride4, const float4 *__restrict__ feat,
    int feat_stride4, int feat_vec4, int row_lo, int row_hi, int4 *__restrict__ rect_sorted,
    float4 *__restrict__ feat_sorted, int64_t *__restrict__ cnt, int64_t *__restrict__ counts,
    int64_t *__restrict__ cnt_live, uint64_t *__restrict__ live_mask,
    int32_t *__restrict__ rank_of) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint64_t key = sorted_keys[r];
    const bool vis = key != ~0ull;
    // the row -> rank inverse (isg_rank_of) while order[r] is at hand
    if (rank_of) rank_of[order[r]] = vis ? (int32_t)r : -1;
    int64_t c = 0, cl = 0;
    uint64_t lm = 0;
    if (vis) {
        const int32_t row = order[r];
        int4 rc = rect[(int64_t)rect_stride4 * row];
        rect_sorted[r] = rc;
        for (int j = 0; j < feat_vec4; j++) feat_sorted[(int64_t)feat_vec4 * r + j] =
            feat[(int64_t)feat_stride4 * row + j];
        int y0 = max(rc.y, row_lo), y1 = min(rc.w, row_hi - 1);
        if (y1 >= y0) c = (int64_t)(rc.z - rc.x + 1) * (int64_t)(y1 - y0 + 1);
        if (r + 1 == n || sorted_keys[r + 1] == ~0ull) counts[0] = r + 1;
        if (cnt_live && c) {
            // live tiles: those some pixel centre of can reach alpha >= 1/255
            // (the rasteriser's conservative box test); a bit mask of them in
            // row-major rect order for rects of <= 64 tiles
            const f32::CullForm cf =
                f32::cull_form(f32::stage(reinterpret_cast<const float *>(feat_sorted), (int)r));
            int k = 0;
            for (int ty = y0; ty <= y1; ty++)
                for (int tx = rc.x; tx <= rc.z; tx++, k++)
                    if (!f32::box_dead_cf(cf, (float)(16 * tx), (float)(16 * ty), 15.0f)) {
                        cl++;
                        if (k < 64) lm |= 1ull << k;
                    }
        }
    } else {
        rect_sorted[r] = make_int4(0, 0, -1, -1);
    }
    if (cnt) cnt[r] = c;
    if (cnt_live) {
        cnt_live[r] = cl;
        if (live_mask) live_mask[r] = lm;
    }
}


// Entry-parallel emission: a block of EMIT_R consecutive ranks owns the
// contiguous slot span [emit_off[r0], emit_off[r0 + EMIT_R]); the block
// stages the ranks' offsets and clipped rects in shared memory and writes the
// span with consecutive threads on consecutive slots (coalesced stores).  Each
// slot finds its rank by a chunked max-scan over the ranks' first slots; its tile is the
// row-major position inside the rank's rect -- the same (tile, rank) pairs in
// the same slots as emit_kernel.
#ifndef EMIT_RANKS
#define EMIT_RANKS 256
#endif
constexpr int EMIT_R = EMIT_RANKS;
constexpr int ECH = 1024;  // slots per scan chunk (4 per thread)

template <typename K, bool CULL>
__global__ void __launch_bounds__(256) emit_span_kernel(int64_t m,
                                                        const int4 *__restrict__ rect_sorted,
                                                        const int64_t *__restrict__ emit_off,
                                                        int tiles_x, int row_lo, int row_hi,
                                                        K *__restrict__ tile_keys,
                                                        int32_t *__restrict__ tile_vals,
                                                        const float *__restrict__ feat_sorted,
                                                        float *__restrict__ partials,
                                                        uint32_t dead_key) {
    __shared__ int64_t soff[EMIT_R + 1];
    __shared__ int4 srect[EMIT_R];
    __shared__ f32::CullForm scf[CULL ? EMIT_R : 1];
    __shared__ int srk[ECH];
    __shared__ int swarp[8];
    const int64_t r0 = (int64_t)blockIdx.x * EMIT_R;
    const int nr = (int)min((int64_t)EMIT_R, m - r0);
    for (int i = threadIdx.x; i <= nr; i += blockDim.x) soff[i] = emit_off[r0 + i];
    for (int i = threadIdx.x; i < nr; i += blockDim.x) {
        int4 rc = rect_sorted[r0 + i];
        rc.y = max(rc.y, row_lo);  // clipped rows, width in .w
        rc.w = rc.z - rc.x + 1;
        srect[i] = rc;
        if (CULL) scf[i] = f32::cull_form(f32::stage(feat_sorted, (int)(r0 + i)));
    }
    __syncthreads();
    const int64_t s0 = soff[0], s1 = soff[nr];
    const uint32_t base_tile = (uint32_t)row_lo * (uint32_t)tiles_x;
    // Each slot's rank: mark every non-empty rank's first slot with its index,
    // then an inclusive max-scan over the chunk (ranks ascend with the slot),
    // instead of a binary search per slot.
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    int carry = -1;  // rank covering the chunk's first slot (from the previous chunk)
    for (int64_t c = s0; c < s1; c += ECH) {
        const int n = (int)min((int64_t)ECH, s1 - c);
        for (int i = t; i < ECH; i += 256) srk[i] = -1;
        __syncthreads();
        for (int i = t; i < nr; i += 256) {
            const int64_t a = soff[i];
            if (soff[i + 1] > a && a >= c && a < c + ECH) srk[a - c] = i;
        }
        __syncthreads();
        int v0 = srk[4 * t], v1 = max(v0, srk[4 * t + 1]), v2 = max(v1, srk[4 * t + 2]),
            v3 = max(v2, srk[4 * t + 3]);
        int x = v3;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x = max(x, y);
        }
        if (lane == 31) swarp[warp] = x;
        __syncthreads();
        int ex = max(carry, __shfl_up_sync(0xffffffffu, x, 1));
        if (lane == 0) ex = carry;
        for (int w = 0; w < warp; w++) ex = max(ex, swarp[w]);
        srk[4 * t] = max(ex, v0);
        srk[4 * t + 1] = max(ex, v1);
        srk[4 * t + 2] = max(ex, v2);
        srk[4 * t + 3] = max(ex, v3);
        __syncthreads();
        for (int i = t; i < n; i += 256) {
            const int64_t o = c + i;
            const int lo = srk[i];
            const int4 rc = srect[lo];
            const int k = (int)(o - soff[lo]);
            const int dy = k / rc.w, dx = k - dy * rc.w;
            uint32_t key = (uint32_t)(rc.y + dy) * (uint32_t)tiles_x - base_tile + (uint32_t)(rc.x + dx);
            if (CULL) {
                const f32::CullForm cf = scf[lo];
                if (f32::box_dead_cf(cf, (float)(16 * (rc.x + dx)), (float)(16 * (rc.y + dy)), 15.0f)) {
                    key = dead_key;
                    float4 *dst = reinterpret_cast<float4 *>(partials + partial_stride<float>() * o);
                    const float4 z = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                    dst[0] = z;
                    dst[1] = z;
                    dst[2] = z;
                }
            }
            tile_keys[o] = (K)key;
            tile_vals[o] = (int32_t)(r0 + lo);
        }
        carry = srk[n - 1];
        __syncthreads();  // srk is rewritten by the next chunk
    }
}

// Thread-per-rank emission of the live lists: each rank writes its live
// (tile, slot) pairs into its own span [live_off[r], live_off[r + 1]) in
// row-major rect order (consecutive ranks' spans are adjacent, so a warp's
// stores stay within one small region).  Rects of <= 64 tiles walk the set
// bits of the rank's live mask; larger ones repeat the box test.
template <typename K>
__global__ void __launch_bounds__(EMIT_T) emit_live_thread_kernel(
    int64_t m, const int4 *__restrict__ rect_sorted, const int64_t *__restrict__ live_off,
    const uint64_t *__restrict__ live_mask, const float *__restrict__ feat_sorted, int tiles_x,
    int row_lo, int row_hi, K *__restrict__ tile_keys, int32_t *__restrict__ slot_rank) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    int64_t out = live_off[r];
    const int64_t end = live_off[r + 1];
    if (out == end) return;
    const int4 rc = rect_sorted[r];
    const int y0 = max(rc.y, row_lo), y1 = min(rc.w, row_hi - 1);
    const int w = rc.z - rc.x + 1;
    const int n = (y1 - y0 + 1) * w;
    const uint32_t base = (uint32_t)(y0 - row_lo) * (uint32_t)tiles_x + (uint32_t)rc.x;
    if (n <= 64) {
        uint64_t mk = live_mask[r];
        while (mk) {
            const int k = __ffsll((long long)mk) - 1;
            mk &= mk - 1;
            const int dy = k / w, dx = k - dy * w;
            tile_keys[out] = (K)(base + (uint32_t)dy * (uint32_t)tiles_x + (uint32_t)dx);
            slot_rank[out] = (int32_t)r;
            out++;
        }
    } else {
        const f32::CullForm cf = f32::cull_form(f32::stage(feat_sorted, (int)r));
        for (int ty = y0; ty <= y1; ty++)
            for (int tx = rc.x; tx <= rc.z; tx++)
                if (!f32::box_dead_cf(cf, (float)(16 * tx), (float)(16 * ty), 15.0f)) {
                    tile_keys[out] = (K)((uint32_t)(ty - row_lo) * (uint32_t)tiles_x +
                                         (uint32_t)tx);
                    slot_rank[out] = (int32_t)r;
                    out++;
                }
    }
}

template <typename K>
__global__ void tile_offsets_kernel(int64_t e, const K *__restrict__ keys, int n_tiles,
                                    int32_t *__restrict__ offsets,
                                    const int64_t *__restrict__ e_dev) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > n_tiles) return;
    if (e_dev) e = min(e, *e_dev);
    int64_t lo = 0, hi = e;  // lower_bound(keys, t)
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if ((uint32_t)keys[mid] < (uint32_t)t) lo = mid + 1;
        else hi = mid;
    }
    offsets[t] = (int32_t)lo;
}

// heavy_pct > 0: only the lists at least heavy_pct % of the mean length are
// ordered heaviest first; the others keep list (row-major) order after them,
// so neighbouring tiles -- which share splats -- still run together (L2 reuse
// of the staged features).  heavy_pct == 0: every list by length.
__global__ void tile_order_keys_kernel(int n_tiles, const int32_t *__restrict__ offsets,
                                       int heavy_pct, uint16_t *__restrict__ keys,
                                       int32_t *__restrict__ vals) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tiles) return;
    const int len = offsets[t + 1] - offsets[t];
    uint16_t k = (uint16_t)(65535 - min(len, 65535));
    if (heavy_pct > 0) {
        const int64_t total = offsets[n_tiles] - offsets[0];
        const bool heavy = (int64_t)len * 100 * n_tiles >= (int64_t)heavy_pct * total;
        k = heavy ? (uint16_t)(32767 - min(len, 32767)) : (uint16_t)65535;
    }
    keys[t] = k;
    vals[t] = t;
}

// Heaviest-first launch order in one CTA (any tile count): tiles bucketed by
// list length into OB linear buckets of width max/OB (longest first), a
// tile's place inside its bucket taken by a shared-memory atomic.  The order
// inside a bucket is arbitrary -- it only schedules CTAs; no result depends
// on it.
constexpr int OB = 1024;
__global__ void __launch_bounds__(1024) tile_order_kernel(int n_tiles,
                                                          const int32_t *__restrict__ offsets,
                                                          int32_t *__restrict__ order) {
    __shared__ int cnt[OB];
    __shared__ int smax;
    if (threadIdx.x == 0) smax = 1;
    for (int b = threadIdx.x; b < OB; b += blockDim.x) cnt[b] = 0;
    __syncthreads();
    int m = 0;
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x)
        m = max(m, offsets[t + 1] - offsets[t]);
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(&smax, m);
    __syncthreads();
    const int64_t mx = (int64_t)smax + 1;
    auto bucket = [&](int len) { return OB - 1 - (int)((int64_t)len * OB / mx); };
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x)
        atomicAdd(&cnt[bucket(offsets[t + 1] - offsets[t])], 1);
    __syncthreads();
    // exclusive scan of the bucket counts (OB == blockDim.x)
    {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        __shared__ int sw[32];
        const int v = cnt[threadIdx.x];
        int x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) sw[warp] = x;
        __syncthreads();
        int before = 0;
        for (int w = 0; w < warp; w++) before += sw[w];
        __syncthreads();
        cnt[threadIdx.x] = before + x - v;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x)
        order[atomicAdd(&cnt[bucket(offsets[t + 1] - offsets[t])], 1)] = t;
}

inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace isg

using namespace isg;

extern "C" int isg_sort_u64(void *workspace, size_t *ws_bytes, const uint64_t *keys_in,
                            uint64_t *keys_out, const int32_t *vals_in, int32_t *vals_out,
                            int64_t n, int32_t begin_bit, int32_t end_bit, void *stream) {
    if (!ws_bytes || n < 0 || n > INT32_MAX || begin_bit < 0 || end_bit > 64 ||
        begin_bit >= end_bit)
        return (int)cudaErrorInvalidValue;
    return radix::sort_pairs<uint64_t>(workspace, ws_bytes, keys_in, keys_out, vals_in, vals_out, n,
                                  begin_bit, end_bit, (cudaStream_t)stream);
}

namespace isg {
#ifndef DEPTH_LO_BIT
#define DEPTH_LO_BIT 24
#endif
constexpr int64_t TIE_INSERTION_MAX = 64;

__device__ __forceinline__ bool kv_less(uint64_t ka, int32_t va, uint64_t kb, int32_t vb) {
    return ka < kb || (ka == kb && va < vb);
}

__device__ void sift_down(uint64_t *k, int32_t *v, int64_t root, int64_t end) {
    while (2 * root + 1 < end) {
        int64_t c = 2 * root + 1;
        if (c + 1 < end && kv_less(k[c], v[c], k[c + 1], v[c + 1])) c++;
        if (!kv_less(k[root], v[root], k[c], v[c])) return;
        const uint64_t tk = k[root];
        const int32_t tv = v[root];
        k[root] = k[c];
        v[root] = v[c];
        k[c] = tk;
        v[c] = tv;
        root = c;
    }
}

__device__ void heap_sort_run(uint64_t *k, int32_t *v, int64_t len) {
    for (int64_t s = len / 2 - 1; s >= 0; s--) sift_down(k, v, s, len);
    for (int64_t e = len - 1; e > 0; e--) {
        const uint64_t tk = k[0];
        const int32_t tv = v[0];
        k[0] = k[e];
        v[0] = v[e];
        k[e] = tk;
        v[e] = tv;
        sift_down(k, v, 0, e);
    }
}

// After a stable sort on key bits [DEPTH_LO_BIT, 64) the only possible
// disorder is inside runs of equal top bits (depths equal to ~2^-(52 -
// DEPTH_LO_BIT) relative).  One thread per run start checks its run and
// insertion-sorts it by the full key (strict comparison: equal keys keep their
// ascending-id order; runs longer than TIE_INSERTION_MAX are heap-sorted by
// (key, id): O(k log k) for any run).  Runs of the culled key ~0 are
// identical and already in id order.
__global__ void __launch_bounds__(256) depth_tie_fix_kernel(int64_t n, uint64_t *keys,
                                                            int32_t *vals) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t k = keys[i];
    if (k == ~0ull) return;
    const uint64_t hi = k >> DEPTH_LO_BIT;
    if (i > 0 && (keys[i - 1] >> DEPTH_LO_BIT) == hi) return;      // not a run start
    if (i + 1 >= n || (keys[i + 1] >> DEPTH_LO_BIT) != hi) return;  // singleton
    int64_t j = i + 1;
    bool sorted = true;
    while (j < n && (keys[j] >> DEPTH_LO_BIT) == hi) {
        if (keys[j] < keys[j - 1]) sorted = false;
        j++;
    }
    if (sorted) return;
    if (j - i <= TIE_INSERTION_MAX) {
        for (int64_t a = i + 1; a < j; a++) {
            const uint64_t key = keys[a];
            const int32_t val = vals[a];
            int64_t b = a - 1;
            while (b >= i && keys[b] > key) {
                keys[b + 1] = keys[b];
                vals[b + 1] = vals[b];
                b--;
            }
            keys[b + 1] = key;
            vals[b + 1] = val;
        }
        return;
    }
    // long run: heapsort by (key, value) -- values are the ascending ids of
    // equal keys, so this is the stable order; O(k log k) worst case
    heap_sort_run(keys + i, vals + i, j - i);
}
}  // namespace isg

// Depth order (np.lexsort((indices, depth)), rasterizer.py:161-163): stable
// radix sort of the float64 depth bits over id-ordered values, in 5 passes of
// the top 40 bits plus the run fix-up -- bit-identical to the full 64-bit sort.
extern "C" int isg_sort_depth(void *workspace, size_t *ws_bytes, const uint64_t *keys_in,
                              uint64_t *keys_out, const int32_t *vals_in, int32_t *vals_out,
                              int64_t n, void *stream) {
    if (!ws_bytes || n < 0 || n > INT32_MAX) return (int)cudaErrorInvalidValue;
    const int e = radix::sort_pairs<uint64_t>(workspace, ws_bytes, keys_in, keys_out, vals_in,
                                              vals_out, n, DEPTH_LO_BIT, 64,
                                              (cudaStream_t)stream);
    if (e != 0 || !workspace || n == 0) return e;
    depth_tie_fix_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(n, keys_out,
                                                                              vals_out);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_sort_u32(void *workspace, size_t *ws_bytes, const uint32_t *keys_in,
                            uint32_t *keys_out, const int32_t *vals_in, int32_t *vals_out,
                            int64_t n, int32_t begin_bit, int32_t end_bit, void *stream) {
    if (!ws_bytes || n < 0 || n > INT32_MAX || begin_bit < 0 || end_bit > 32 ||
        begin_bit >= end_bit)
        return (int)cudaErrorInvalidValue;
    return radix::sort_pairs<uint32_t>(workspace, ws_bytes, keys_in, keys_out, vals_in, vals_out, n,
                                  begin_bit, end_bit, (cudaStream_t)stream);
}

extern "C" int isg_tile_order(int32_t n_tiles, const int32_t *offsets, int32_t *order,
                              void *stream) {
    if (n_tiles < 0 || (n_tiles > 0 && (!offsets || !order))) return (int)cudaErrorInvalidValue;
    if (n_tiles == 0) return 0;
    tile_order_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(n_tiles, offsets, order);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_tile_order_keys(int32_t n_tiles, const int32_t *offsets, int32_t heavy_pct,
                                   uint16_t *keys16, int32_t *vals, void *stream) {
    if (n_tiles < 0 || (n_tiles > 0 && (!offsets || !keys16 || !vals)))
        return (int)cudaErrorInvalidValue;
    if (n_tiles == 0) return 0;
    tile_order_keys_kernel<<<blocks_for(n_tiles, 256), 256, 0, (cudaStream_t)stream>>>(
        n_tiles, offsets, heavy_pct, keys16, vals);
    ISG_CHECK_LAUNCH();
    return 0;
}

static int bin_count(void *workspace, size_t *ws_bytes, int64_t n, const uint64_t *sorted_keys,
                     const int32_t *order, const int4 *rect, int rect_stride4,
                     const float4 *feat, int feat_stride4, int vec4, int32_t row_lo,
                     int32_t row_hi, int32_t *rect_sorted, void *feat_sorted, int64_t *emit_off,
                     int64_t *counts, void *stream, bool live = false,
                     int64_t *live_off = nullptr, uint64_t *live_mask = nullptr,
                     bool full_offsets = true, int32_t *rank_of = nullptr) {
    if (!ws_bytes || n < 0 || n > INT32_MAX || row_lo < 0 || row_hi < row_lo)
        return (int)cudaErrorInvalidValue;
    const size_t scan_bytes = scan_i64_ws_bytes(n > 0 ? n : 1);
    const size_t cnt_bytes = align_up(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    const size_t need = (live ? 2 : 1) * cnt_bytes + align_up(scan_bytes);
    if (!workspace) {
        *ws_bytes = need;
        return 0;
    }
    if (*ws_bytes < need || (live && (!live_off || !live_mask))) return (int)cudaErrorInvalidValue;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(counts, 0, (live ? 3 : 2) * sizeof(int64_t), s);
    if (e != cudaSuccess) return (int)e;
    if (full_offsets) e = cudaMemsetAsync(emit_off, 0, sizeof(int64_t), s);
    if (e == cudaSuccess && live_off) e = cudaMemsetAsync(live_off, 0, sizeof(int64_t), s);
    if (e != cudaSuccess) return (int)e;
    if (n == 0) return 0;
    int64_t *cnt = (int64_t *)workspace;
    int64_t *cnt_live = live_off ? (int64_t *)((char *)workspace + cnt_bytes) : nullptr;
    void *scan_ws = (char *)workspace + (live_off ? 2 : 1) * cnt_bytes;
    gather_rank_kernel<<<blocks_for(n, GATHER_T), GATHER_T, 0, s>>>(
        n, sorted_keys, order, rect, rect_stride4, feat, feat_stride4, vec4, row_lo, row_hi,
        (int4 *)rect_sorted, (float4 *)feat_sorted, full_offsets ? cnt : nullptr, counts,
        cnt_live, live_mask, rank_of);
    ISG_CHECK_LAUNCH();
    int se = 0;
    if (full_offsets) {
        se = scan_i64(scan_ws, scan_bytes, n, cnt, emit_off, counts + 1, s);
        if (se != 0) return se;
    }
    if (live_off) {
        se = scan_i64(scan_ws, scan_bytes, n, cnt_live, live_off, counts + 2, s);
        if (se != 0) return se;
    }
    return 0;
}

extern "C" int isg_bin_count(void *workspace, size_t *ws_bytes, int64_t n,
                             const uint64_t *sorted_keys, const int32_t *order,
                             const int32_t *rect, const void *feat, int32_t feat_dtype,
                             int32_t row_lo, int32_t row_hi, int32_t *rect_sorted,
                             void *feat_sorted, int64_t *emit_off, int64_t *counts,
                             void *stream) {
    const int vec4 = feat_dtype == ISG_F64 ? 6 : 3;  // 12 values per splat
    return bin_count(workspace, ws_bytes, n, sorted_keys, order, (const int4 *)rect, 1,
                     (const float4 *)feat, vec4, vec4, row_lo, row_hi, rect_sorted, feat_sorted,
                     emit_off, counts, stream);
}

extern "C" int isg_bin_count_live(void *workspace, size_t *ws_bytes, int64_t n,
                                  const uint64_t *sorted_keys, const int32_t *order,
                                  const int32_t *rect, const int32_t *payload, const float *feat,
                                  int32_t row_lo, int32_t row_hi, int32_t *rect_sorted,
                                  float *feat_sorted, int64_t *emit_off, int64_t *live_off,
                                  uint64_t *live_mask, int64_t *counts, void *stream) {
    const int4 *p = (const int4 *)payload;
    if (payload)  // 64-byte payload rows: rect then the 12 float32 features
        return bin_count(workspace, ws_bytes, n, sorted_keys, order, p, 4, (const float4 *)(p + 1),
                         4, 3, row_lo, row_hi, rect_sorted, feat_sorted, emit_off, counts, stream,
                         true, live_off, live_mask);
    return bin_count(workspace, ws_bytes, n, sorted_keys, order, (const int4 *)rect, 1,
                     (const float4 *)feat, 3, 3, row_lo, row_hi, rect_sorted, feat_sorted,
                     emit_off, counts, stream, true, live_off, live_mask);
}

extern "C" int isg_bin_count_train(void *workspace, size_t *ws_bytes, int64_t n,
                                   const uint64_t *sorted_keys, const int32_t *order,
                                   const int32_t *rect, const float *feat, int32_t row_lo,
                                   int32_t row_hi, int32_t *rect_sorted, float *feat_sorted,
                                   int64_t *live_off, uint64_t *live_mask, int32_t *rank_of,
                                   int64_t *counts, void *stream) {
    if (workspace && (!live_off || !live_mask)) return (int)cudaErrorInvalidValue;
    return bin_count(workspace, ws_bytes, n, sorted_keys, order, (const int4 *)rect, 1,
                     (const float4 *)feat, 3, 3, row_lo, row_hi, rect_sorted, feat_sorted, nullptr,
                     counts, stream, true, live_off, live_mask, false, rank_of);
}

extern "C" int isg_bin_emit_live(int64_t m, const int32_t *rect_sorted, const int64_t *emit_off,
                                 const int64_t *live_off, const uint64_t *live_mask,
                                 const float *feat_sorted, int32_t tiles_x, int32_t row_lo,
                                 int32_t row_hi, void *tile_keys, int32_t key_bytes,
                                 int32_t *slot_rank, void *stream) {
    const int64_t nt = (int64_t)(row_hi - row_lo) * tiles_x;
    if (m < 0 || tiles_x <= 0 || (key_bytes != 2 && key_bytes != 4) ||
        (key_bytes == 2 && nt > 65536) ||
        (m > 0 && (!rect_sorted || !emit_off || !live_off || !live_mask || !feat_sorted ||
                   !tile_keys || !slot_rank)))
        return (int)cudaErrorInvalidValue;
    if (m == 0) return 0;
    if (key_bytes == 2)
        emit_live_thread_kernel<uint16_t><<<blocks_for(m, EMIT_T), EMIT_T, 0, (cudaStream_t)stream>>>(
            m, (const int4 *)rect_sorted, live_off, live_mask, feat_sorted, tiles_x, row_lo,
            row_hi, (uint16_t *)tile_keys, slot_rank);
    else
        emit_live_thread_kernel<uint32_t><<<blocks_for(m, EMIT_T), EMIT_T, 0, (cudaStream_t)stream>>>(
            m, (const int4 *)rect_sorted, live_off, live_mask, feat_sorted, tiles_x, row_lo,
            row_hi, (uint32_t *)tile_keys, slot_rank);

    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_bin_count_rows(void *workspace, size_t *ws_bytes, int64_t n,
                                  const uint64_t *sorted_keys, const int32_t *order,
                                  const int32_t *payload, int32_t row_lo, int32_t row_hi,
                                  int32_t *rect_sorted, float *feat_sorted, int64_t *emit_off,
                                  int64_t *counts, void *stream) {
    // 64-byte payload rows: rect (4 x int32) then the 12 float32 features
    const int4 *p = (const int4 *)payload;
    return bin_count(workspace, ws_bytes, n, sorted_keys, order, p, 4,
                     (const float4 *)(p ? p + 1 : nullptr), 4, 3, row_lo, row_hi, rect_sorted,
                     feat_sorted, emit_off, counts, stream);
}

namespace isg {
// rank_of[order[r]] = r for visible ranks (sorted key != ~0), -1 otherwise:
// the row -> rank inverse that lets row-parallel kernels read rank-ordered
// per-splat data.  order is a permutation, so every row is written.
__global__ void __launch_bounds__(256) rank_of_kernel(int64_t n,
                                                      const uint64_t *__restrict__ sorted_keys,
                                                      const int32_t *__restrict__ order,
                                                      int32_t *__restrict__ rank_of) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    rank_of[order[r]] = sorted_keys[r] != ~0ull ? (int32_t)r : -1;
}
}  // namespace isg

extern "C" int isg_rank_of(int64_t n, const uint64_t *sorted_keys, const int32_t *order,
                           int32_t *rank_of, void *stream) {
    if (n < 0 || n > INT32_MAX || (n > 0 && (!sorted_keys || !order || !rank_of)))
        return (int)cudaErrorInvalidValue;
    if (n == 0) return 0;
    rank_of_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(n, sorted_keys, order,
                                                                        rank_of);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_bin_emit(int64_t m, const int32_t *rect_sorted, const int64_t *emit_off,
                            int32_t tiles_x, int32_t row_lo, int32_t row_hi, uint32_t *tile_keys,
                            int32_t *tile_vals, void *stream) {
    if (m < 0 || tiles_x <= 0) return (int)cudaErrorInvalidValue;
    if (m == 0) return 0;
    emit_span_kernel<uint32_t, false><<<blocks_for(m, EMIT_R), 256, 0, (cudaStream_t)stream>>>(
        m, (const int4 *)rect_sorted, emit_off, tiles_x, row_lo, row_hi, tile_keys, tile_vals,
        nullptr, nullptr, 0u);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_bin_emit16(int64_t m, const int32_t *rect_sorted, const int64_t *emit_off,
                              int32_t tiles_x, int32_t row_lo, int32_t row_hi,
                              uint16_t *tile_keys, int32_t *tile_vals, void *stream) {
    if (m < 0 || tiles_x <= 0 || (int64_t)(row_hi - row_lo) * tiles_x > 65536)
        return (int)cudaErrorInvalidValue;
    if (m == 0) return 0;
    emit_span_kernel<uint16_t, false><<<blocks_for(m, EMIT_R), 256, 0, (cudaStream_t)stream>>>(
        m, (const int4 *)rect_sorted, emit_off, tiles_x, row_lo, row_hi, tile_keys, tile_vals,
        nullptr, nullptr, 0u);
    ISG_CHECK_LAUNCH();
    return 0;
}


extern "C" int isg_sort_u16(void *workspace, size_t *ws_bytes, const uint16_t *keys_in,
                            uint16_t *keys_out, const int32_t *vals_in, int32_t *vals_out,
                            int64_t n, int32_t begin_bit, int32_t end_bit, void *stream) {
    if (!ws_bytes || n < 0 || n > INT32_MAX || begin_bit < 0 || end_bit > 16 ||
        begin_bit >= end_bit)
        return (int)cudaErrorInvalidValue;
    return radix::sort_pairs<uint16_t>(workspace, ws_bytes, keys_in, keys_out, vals_in, vals_out, n,
                                  begin_bit, end_bit, (cudaStream_t)stream);
}

extern "C" int isg_sort_pairs_dev(void *workspace, size_t *ws_bytes, int32_t key_bytes,
                                  const void *keys_in, void *keys_out, const int32_t *vals_in,
                                  int32_t *vals_out, int64_t n_max, const int64_t *n_dev,
                                  int32_t begin_bit, int32_t end_bit, void *stream) {
    if (!ws_bytes || n_max < 0 || n_max > INT32_MAX || begin_bit < 0 || begin_bit >= end_bit ||
        end_bit > 8 * key_bytes)
        return (int)cudaErrorInvalidValue;
    cudaStream_t s = (cudaStream_t)stream;
    if (key_bytes == 2)
        return radix::sort_pairs<uint16_t>(workspace, ws_bytes, (const uint16_t *)keys_in,
                                           (uint16_t *)keys_out, vals_in, vals_out, n_max,
                                           begin_bit, end_bit, s, n_dev);
    if (key_bytes == 4)
        return radix::sort_pairs<uint32_t>(workspace, ws_bytes, (const uint32_t *)keys_in,
                                           (uint32_t *)keys_out, vals_in, vals_out, n_max,
                                           begin_bit, end_bit, s, n_dev);
    if (key_bytes == 8)
        return radix::sort_pairs<uint64_t>(workspace, ws_bytes, (const uint64_t *)keys_in,
                                           (uint64_t *)keys_out, vals_in, vals_out, n_max,
                                           begin_bit, end_bit, s, n_dev);
    return (int)cudaErrorInvalidValue;
}

extern "C" int isg_tile_offsets_dev(int64_t e_max, const int64_t *e_dev, const void *sorted_keys,
                                    int32_t key_bytes, int32_t n_tiles, int32_t *offsets,
                                    void *stream) {
    if (e_max < 0 || n_tiles < 0 || !offsets || (key_bytes != 2 && key_bytes != 4) ||
        (key_bytes == 2 && n_tiles > 65536))
        return (int)cudaErrorInvalidValue;
    if (key_bytes == 2)
        tile_offsets_kernel<uint16_t><<<blocks_for(n_tiles + 1, 256), 256, 0,
                                        (cudaStream_t)stream>>>(
            e_max, (const uint16_t *)sorted_keys, n_tiles, offsets, e_dev);
    else
        tile_offsets_kernel<uint32_t><<<blocks_for(n_tiles + 1, 256), 256, 0,
                                        (cudaStream_t)stream>>>(
            e_max, (const uint32_t *)sorted_keys, n_tiles, offsets, e_dev);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_tile_offsets16(int64_t e, const uint16_t *sorted_tile_keys, int32_t n_tiles,
                                  int32_t *offsets, void *stream) {
    if (e < 0 || n_tiles < 0 || n_tiles > 65536) return (int)cudaErrorInvalidValue;
    tile_offsets_kernel<uint16_t><<<blocks_for(n_tiles + 1, 256), 256, 0, (cudaStream_t)stream>>>(
        e, sorted_tile_keys, n_tiles, offsets, nullptr);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_tile_offsets(int64_t e, const uint32_t *sorted_tile_keys, int32_t n_tiles,
                                int32_t *offsets, void *stream) {
    if (e < 0 || n_tiles < 0) return (int)cudaErrorInvalidValue;
    tile_offsets_kernel<<<blocks_for(n_tiles + 1, 256), 256, 0, (cudaStream_t)stream>>>(
        e, sorted_tile_keys, n_tiles, offsets, (const int64_t *)nullptr);
    ISG_CHECK_LAUNCH();
    return 0;
}
