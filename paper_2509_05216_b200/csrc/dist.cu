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
#include <cub/cub.cuh>

#include "common.cuh"

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

__global__ void route_count_kernel(int64_t n, const uint8_t *__restrict__ flag,
                                   const int4 *__restrict__ rect, Bands bands,
                                   int64_t *__restrict__ cnt, int32_t *__restrict__ dlo) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t c = 0;
    int lo = 0;
    if (flag[i]) {
        const int4 rc = rect[i];
        lo = band_of(bands, rc.y);
        const int hi = band_of(bands, rc.w);
        c = hi - lo + 1;
    }
    cnt[i] = c;
    dlo[i] = lo;
}

__global__ void route_emit_kernel(int64_t n, const int64_t *__restrict__ off,
                                  const int32_t *__restrict__ dlo, uint32_t *__restrict__ keys,
                                  int32_t *__restrict__ vals) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t o = off[i], c = off[i + 1] - o;
    for (int64_t k = 0; k < c; k++) {
        keys[o + k] = (uint32_t)(dlo[i] + k);
        vals[o + k] = (int32_t)i;
    }
}

// record: [key lo, key hi, gid, 0, rect x4, feat x12] as 20 x 32-bit words
__global__ void route_gather_kernel(int64_t s, const int32_t *__restrict__ rows,
                                    const uint64_t *__restrict__ key, const int4 *__restrict__ rect,
                                    const int4 *__restrict__ feat, int64_t id_base,
                                    int4 *__restrict__ rec) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= s) return;
    const int64_t i = rows[k];
    const uint64_t kk = key[i];
    int4 *r = rec + 5 * k;
    r[0] = make_int4((int)(uint32_t)kk, (int)(uint32_t)(kk >> 32), (int)(id_base + i), 0);
    r[1] = rect[i];
    r[2] = feat[3 * i];
    r[3] = feat[3 * i + 1];
    r[4] = feat[3 * i + 2];
}

__global__ void unpack_kernel(int64_t r, const int4 *__restrict__ rec, uint64_t *__restrict__ key,
                              int32_t *__restrict__ gid, int4 *__restrict__ rect,
                              int4 *__restrict__ feat) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= r) return;
    const int4 *p = rec + 5 * k;
    const int4 h = p[0];
    key[k] = (uint64_t)(uint32_t)h.x | ((uint64_t)(uint32_t)h.y << 32);
    gid[k] = h.z;
    rect[k] = p[1];
    feat[3 * k] = p[2];
    feat[3 * k + 1] = p[3];
    feat[3 * k + 2] = p[4];
}

__global__ void block_count_kernel(int64_t m, const int4 *__restrict__ rect_sorted, int row_lo,
                                   int row_hi, int canon, int64_t *__restrict__ nb) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    const int4 rc = rect_sorted[r];
    const int y0 = max(rc.y, row_lo), y1 = min(rc.w, row_hi - 1);
    nb[r] = y1 >= y0 ? (int64_t)(y1 / canon - y0 / canon + 1) : 0;
}

struct Shards {
    int n;
    int64_t start[MAX_BANDS + 1];  // global id boundaries of the Gaussian shards
};

__device__ __forceinline__ int shard_of(const Shards &s, int64_t gid) {
    int lo = 0, hi = s.n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s.start[mid] <= gid) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Per rank r: fold its slots [emit_off[r], emit_off[r+1]) per canonical block
// (float64) into records rec_off[r] + b: owner shard (sort key), owner-local
// row and the 9 block sums.
template <typename T>
__global__ void block_fold_kernel(int64_t m, const int64_t *__restrict__ emit_off,
                                  const T *__restrict__ partials,
                                  const int4 *__restrict__ rect_sorted, int row_lo, int row_hi,
                                  int canon, const int64_t *__restrict__ rec_off,
                                  const int32_t *__restrict__ order,
                                  const int32_t *__restrict__ gid, Shards shards,
                                  uint32_t *__restrict__ rec_owner, int32_t *__restrict__ rec_row,
                                  double *__restrict__ rec_val) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    const int4 rc = rect_sorted[r];
    const int y0 = max(rc.y, row_lo), y1 = min(rc.w, row_hi - 1);
    if (y1 < y0) return;
    const int64_t p0 = emit_off[r], w = rc.z - rc.x + 1;
    const int64_t g = gid[order[r]];
    const int owner = shard_of(shards, g);
    const int32_t row = (int32_t)(g - shards.start[owner]);
    int64_t o = rec_off[r];
    for (int b = y0 / canon; b <= y1 / canon; b++, o++) {
        const int ys = max(y0, b * canon), ye = min(y1, b * canon + canon - 1);
        double bs[9];
#pragma unroll
        for (int k = 0; k < 9; k++) bs[k] = 0.0;
        for (int64_t p = p0 + (ys - y0) * w; p < p0 + (ye - y0 + 1) * w; p++) {
            const T *src = partials + partial_stride<T>() * p;
#pragma unroll
            for (int k = 0; k < 9; k++) bs[k] += (double)src[k];
        }
        rec_owner[o] = (uint32_t)owner;
        rec_row[o] = row;
        double *dst = rec_val + 9 * o;
#pragma unroll
        for (int k = 0; k < 9; k++) dst[k] = bs[k];
    }
}

// grad record: [row, 0, 9 doubles] = 20 words
__global__ void grad_gather_kernel(int64_t s, const int32_t *__restrict__ idx,
                                   const int32_t *__restrict__ rec_row,
                                   const double *__restrict__ rec_val, int32_t *__restrict__ out) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= s) return;
    const int64_t i = idx[k];
    int32_t *o = out + 20 * k;
    o[0] = rec_row[i];
    o[1] = 0;
    double *d = reinterpret_cast<double *>(o + 2);
#pragma unroll
    for (int q = 0; q < 9; q++) d[q] = rec_val[9 * i + q];
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

__global__ void scan_finish_kernel(int64_t n, const int64_t *__restrict__ off,
                                   int64_t *__restrict__ total) {
    total[0] = off[n];
}

inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace isg

using namespace isg;

// Exclusive scan of n int64 counts into off[0..n] (off[0] = 0) and *total.
extern "C" int isg_scan_i64(void *workspace, size_t *ws_bytes, int64_t n, const int64_t *cnt,
                            int64_t *off, int64_t *total, void *stream) {
    if (!ws_bytes || n < 0 || n > INT32_MAX) return (int)cudaErrorInvalidValue;
    size_t need = 0;
    cub::DeviceScan::InclusiveSum(nullptr, need, (const int64_t *)nullptr, (int64_t *)nullptr,
                                  (int)(n > 0 ? n : 1));
    need = al(need);
    if (!workspace) {
        *ws_bytes = need;
        return 0;
    }
    if (*ws_bytes < need) return (int)cudaErrorInvalidValue;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(off, 0, sizeof(int64_t), s);
    if (e != cudaSuccess) return (int)e;
    if (n > 0) {
        e = cub::DeviceScan::InclusiveSum(workspace, need, cnt, off + 1, (int)n, s);
        if (e != cudaSuccess) return (int)e;
    }
    if (total) {
        scan_finish_kernel<<<1, 1, 0, s>>>(n, off, total);
        ISG_CHECK_LAUNCH();
    }
    return 0;
}

static int fill_bands(Bands &b, const int32_t *band_rows, int32_t n_bands) {
    if (n_bands < 1 || n_bands > MAX_BANDS || !band_rows) return 1;
    b.n = n_bands;
    for (int i = 0; i <= n_bands; i++) b.start[i] = band_rows[i];
    return 0;
}

extern "C" int isg_route_count(int64_t n, const uint8_t *flag, const int32_t *rect,
                               const int32_t *band_rows, int32_t n_bands, int64_t *cnt,
                               int32_t *dlo, void *stream) {
    Bands b;
    if (n < 0 || fill_bands(b, band_rows, n_bands)) return (int)cudaErrorInvalidValue;
    if (n == 0) return 0;
    route_count_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
        n, flag, (const int4 *)rect, b, cnt, dlo);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_route_emit(int64_t n, const int64_t *off, const int32_t *dlo, uint32_t *keys,
                              int32_t *vals, void *stream) {
    if (n < 0) return (int)cudaErrorInvalidValue;
    if (n == 0) return 0;
    route_emit_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(n, off, dlo, keys,
                                                                            vals);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_route_gather(int64_t s, const int32_t *rows, const uint64_t *key,
                                const int32_t *rect, const float *feat, int64_t id_base,
                                int32_t *records, void *stream) {
    if (s < 0) return (int)cudaErrorInvalidValue;
    if (s == 0) return 0;
    route_gather_kernel<<<blocks_for(s, 256), 256, 0, (cudaStream_t)stream>>>(
        s, rows, key, (const int4 *)rect, (const int4 *)feat, id_base, (int4 *)records);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_records_unpack(int64_t r, const int32_t *records, uint64_t *key, int32_t *gid,
                                  int32_t *rect, float *feat, void *stream) {
    if (r < 0) return (int)cudaErrorInvalidValue;
    if (r == 0) return 0;
    unpack_kernel<<<blocks_for(r, 256), 256, 0, (cudaStream_t)stream>>>(
        r, (const int4 *)records, key, gid, (int4 *)rect, (int4 *)feat);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_block_count(int64_t m, const int32_t *rect_sorted, int32_t row_lo,
                               int32_t row_hi, int32_t canon_rows, int64_t *nb, void *stream) {
    if (m < 0 || canon_rows < 1) return (int)cudaErrorInvalidValue;
    if (m == 0) return 0;
    block_count_kernel<<<blocks_for(m, 256), 256, 0, (cudaStream_t)stream>>>(
        m, (const int4 *)rect_sorted, row_lo, row_hi, canon_rows, nb);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_block_fold(int32_t feat_dtype, int64_t m, const int64_t *emit_off,
                              const void *partials, const int32_t *rect_sorted, int32_t row_lo,
                              int32_t row_hi, int32_t canon_rows, const int64_t *rec_off,
                              const int32_t *order, const int32_t *gid,
                              const int64_t *shard_start, int32_t n_shards, uint32_t *rec_owner,
                              int32_t *rec_row, double *rec_val, void *stream) {
    if (m < 0 || canon_rows < 1 || n_shards < 1 || n_shards > MAX_BANDS || !shard_start)
        return (int)cudaErrorInvalidValue;
    if (m == 0) return 0;
    Shards sh;
    sh.n = n_shards;
    for (int i = 0; i <= n_shards; i++) sh.start[i] = shard_start[i];
    cudaStream_t s = (cudaStream_t)stream;
    const int4 *rs = (const int4 *)rect_sorted;
    if (feat_dtype == ISG_F32)
        block_fold_kernel<float><<<blocks_for(m, 256), 256, 0, s>>>(
            m, emit_off, (const float *)partials, rs, row_lo, row_hi, canon_rows, rec_off, order,
            gid, sh, rec_owner, rec_row, rec_val);
    else if (feat_dtype == ISG_F64)
        block_fold_kernel<double><<<blocks_for(m, 256), 256, 0, s>>>(
            m, emit_off, (const double *)partials, rs, row_lo, row_hi, canon_rows, rec_off, order,
            gid, sh, rec_owner, rec_row, rec_val);
    else
        return (int)cudaErrorInvalidValue;
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_grad_gather(int64_t s, const int32_t *idx, const int32_t *rec_row,
                               const double *rec_val, int32_t *out, void *stream) {
    if (s < 0) return (int)cudaErrorInvalidValue;
    if (s == 0) return 0;
    grad_gather_kernel<<<blocks_for(s, 256), 256, 0, (cudaStream_t)stream>>>(s, idx, rec_row,
                                                                             rec_val, out);
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
