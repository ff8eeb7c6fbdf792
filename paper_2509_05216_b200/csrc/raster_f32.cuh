// raster_f32.cuh -- launchers of the float32 production rasteriser
// (raster_f32.cu), dispatched from the C ABI in raster_f64.cu.
#pragma once
// cmask (optional): the forward's per-(tile, quadrant, batch of 32 entries)
// contribution masks, 4 * (E / 32 + n_tiles + 1) words; the backward given
// the same array walks only the entries some pixel composited.
// tile_order (optional): CTA b processes list position tile_order[b] (the
// launch order, e.g. heaviest tiles first); results do not depend on it.
// slot_rank (optional): the lists hold live-only subtotal slots (entry ->
// rank through slot_rank); the backward writes each entry's record at its
// slot with the tile row in float 9 (isg_bin_emit_live layout).
#include <cuda_runtime.h>
#include <stdint.h>

#include "isogs.h"

namespace isg {

// Backward list chunking (isg_chunks, isogs.h).
using ChunkArgs = isg_chunks;

void launch_raster_fwd_f32(int n_tiles, int W, int H, int tiles_x, int row_lo,
                           const int32_t *tile_ids, const int32_t *tile_order,
                           const int32_t *offsets, const int32_t *entries,
                           const float *feat, float bg0, float bg1, float bg2, void *image,
                           int image_f64, float *t_final, int32_t *n_last, int32_t *n_contrib,
                           int32_t *n_iter, int64_t *touched, uint32_t *cmask,
                           const ChunkArgs *chunks, const int32_t *slot_rank, cudaStream_t s);

template <typename DL>
void launch_raster_bwd_f32(int n_tiles, int W, int H, int tiles_x, int row_lo,
                           const int32_t *tile_ids, const int32_t *tile_order,
                           const int32_t *offsets, const int32_t *entries,
                           const float *feat, const int4 *rect_sorted, const int64_t *emit_off,
                           float bg0, float bg1, float bg2, const float *t_final,
                           const int32_t *n_last, const DL *dl, float *partials,
                           const uint32_t *cmask, const ChunkArgs *chunks,
                           const int32_t *slot_rank, cudaStream_t s);

}  // namespace isg
