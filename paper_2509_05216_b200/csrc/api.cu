// api.cu -- device glue of the reference-compatible render API
// (paper_2509_05216_b200/rasterizer.py): the stable compaction of projected
// rows into SplatBatch columns (rasterizer.py:142-158 `keep`) and the
// depth-ordered gather of those columns into raster features
// (rasterizer.py:294-345), one kernel each instead of a chain of framework
// indexing ops over millions of rows.
#include <stdint.h>

#include "common.cuh"
#include "radix.cuh"

namespace isg {

__global__ void flag_count_kernel(int64_t n, const uint8_t *__restrict__ flag,
                                  int64_t *__restrict__ cnt) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) cnt[i] = flag[i] ? 1 : 0;
}

struct BatchCols {
    double *mean2d, *cov2d, *conic, *depth, *color, *opacity;
    int32_t *tile_min, *tile_max;
    int64_t *indices;
};

// Row i (kept) -> column position pos[i] (the exclusive scan of the keep
// flags: kept rows in ascending order, like full[keep]).
__global__ void compact_batch_kernel(int64_t n, const uint8_t *__restrict__ flag,
                                     const int64_t *__restrict__ pos,
                                     const double *__restrict__ full64,
                                     const int4 *__restrict__ rect,
                                     const int64_t *__restrict__ indices, BatchCols o) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !flag[i]) return;
    const int64_t p = pos[i];
    const double *f = full64 + 16 * i;
    o.mean2d[2 * p] = f[0];
    o.mean2d[2 * p + 1] = f[1];
    for (int k = 0; k < 3; k++) {
        o.cov2d[3 * p + k] = f[2 + k];
        o.conic[3 * p + k] = f[5 + k];
        o.color[3 * p + k] = f[9 + k];
    }
    o.depth[p] = f[8];
    o.opacity[p] = f[12];
    const int4 rc = rect[i];
    o.tile_min[2 * p] = rc.x;
    o.tile_min[2 * p + 1] = rc.y;
    o.tile_max[2 * p] = rc.z;
    o.tile_max[2 * p + 1] = rc.w;
    o.indices[p] = indices ? indices[i] : i;
}

// Sorted row r <- batch row order[r]: the 12 raster features (mean2d,
// conic, opacity, colour, 3 pads) converted to F, and the tile rect.
template <typename F>
__global__ void gather_batch_kernel(int64_t m, const int64_t *__restrict__ order,
                                    const double *__restrict__ mean2d,
                                    const double *__restrict__ conic,
                                    const double *__restrict__ color,
                                    const double *__restrict__ opacity,
                                    const int32_t *__restrict__ tile_min,
                                    const int32_t *__restrict__ tile_max, F *__restrict__ feat,
                                    int4 *__restrict__ rect) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    const int64_t i = order[r];
    F *o = feat + 12 * r;
    o[0] = (F)mean2d[2 * i];
    o[1] = (F)mean2d[2 * i + 1];
    o[2] = (F)conic[3 * i];
    o[3] = (F)conic[3 * i + 1];
    o[4] = (F)conic[3 * i + 2];
    o[5] = (F)opacity[i];
    o[6] = (F)color[3 * i];
    o[7] = (F)color[3 * i + 1];
    o[8] = (F)color[3 * i + 2];
    o[9] = o[10] = o[11] = (F)0;
    rect[r] = make_int4(tile_min[2 * i], tile_min[2 * i + 1], tile_max[2 * i], tile_max[2 * i + 1]);
}

}  // namespace isg

using namespace isg;

extern "C" int isg_compact_count(void *workspace, size_t *ws_bytes, int64_t n,
                                 const uint8_t *flag, int64_t *pos, void *stream) {
    if (!ws_bytes || n < 0 || n > INT32_MAX) return (int)cudaErrorInvalidValue;
    const size_t scan_bytes = (scan_i64_ws_bytes(n > 0 ? n : 1) + 255) & ~(size_t)255;
    const size_t need = scan_bytes + sizeof(int64_t) * (size_t)(n > 0 ? n : 1);
    if (!workspace) {
        *ws_bytes = need;
        return 0;
    }
    if (*ws_bytes < need || !pos || (n > 0 && !flag)) return (int)cudaErrorInvalidValue;
    cudaStream_t s = (cudaStream_t)stream;
    if (n == 0) return (int)cudaMemsetAsync(pos, 0, sizeof(int64_t), s);
    int64_t *cnt = (int64_t *)((char *)workspace + scan_bytes);
    flag_count_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, flag, cnt);
    ISG_CHECK_LAUNCH();
    return scan_i64(workspace, scan_bytes, n, cnt, pos, nullptr, s);
}

extern "C" int isg_compact_batch(int64_t n, const uint8_t *flag, const int64_t *pos,
                                 const double *full64, const int32_t *rect,
                                 const int64_t *indices, double *mean2d, double *cov2d,
                                 double *conic, double *depth, double *color, double *opacity,
                                 int32_t *tile_min, int32_t *tile_max, int64_t *indices_out,
                                 void *stream) {
    if (n < 0 || (n > 0 && (!flag || !pos || !full64 || !rect || !indices_out)))
        return (int)cudaErrorInvalidValue;
    if (n == 0) return 0;
    BatchCols o{mean2d, cov2d, conic, depth, color, opacity, tile_min, tile_max, indices_out};
    compact_batch_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
        n, flag, pos, full64, (const int4 *)rect, indices, o);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_gather_batch(int64_t m, const int64_t *order, const double *mean2d,
                                const double *conic, const double *color, const double *opacity,
                                const int32_t *tile_min, const int32_t *tile_max,
                                int32_t feat_dtype, void *feat, int32_t *rect, void *stream) {
    if (m < 0 || (feat_dtype != ISG_F32 && feat_dtype != ISG_F64) ||
        (m > 0 && (!order || !mean2d || !conic || !color || !opacity || !tile_min ||
                   !tile_max || !feat || !rect)))
        return (int)cudaErrorInvalidValue;
    if (m == 0) return 0;
    cudaStream_t s = (cudaStream_t)stream;
    if (feat_dtype == ISG_F32)
        gather_batch_kernel<float><<<blocks_for(m, 256), 256, 0, s>>>(
            m, order, mean2d, conic, color, opacity, tile_min, tile_max, (float *)feat,
            (int4 *)rect);
    else
        gather_batch_kernel<double><<<blocks_for(m, 256), 256, 0, s>>>(
            m, order, mean2d, conic, color, opacity, tile_min, tile_max, (double *)feat,
            (int4 *)rect);
    ISG_CHECK_LAUNCH();
    return 0;
}
