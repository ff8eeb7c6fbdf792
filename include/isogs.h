/*
 * isogs.h -- C ABI of the B200 training-step hot path (libisogs.so).
 *
 * Drop-in boundary for the numba kernels of the reference package
 * (isosplat 0.1.0; paths relative to /root/reference/pkg/src/isosplat/).
 * Every entry point:
 *   - takes DEVICE pointers, element counts, POD structs and a cudaStream_t
 *     (passed as void*); no torch or C++ types cross the boundary;
 *   - never allocates: the caller owns every buffer, including workspaces
 *     whose size is queried first (two-phase, CUB style);
 *   - returns 0 (cudaSuccess) or a cudaError_t code (cudaErrorInvalidValue = 1
 *     for bad arguments); it never aborts or exits;
 *   - is reentrant and stream ordered (no global mutable state), so one host
 *     thread or process per GPU can drive it concurrently.
 * Floating-point "dtype" tags select the kernel instantiation, mirroring the
 * reference's `dtype` argument: ISG_F32 (production) or ISG_F64 (tight
 * cross-check build).
 */
#ifndef ISOGS_H
#define ISOGS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ISG_F32 0
#define ISG_F64 1
#define ISG_TILE 16

/* Pinhole camera (camera.py:15-54): q = R p + t, u = fx q.x / q.z + cx.
 * C = -R^T t is the camera centre (Camera.position). */
typedef struct isg_camera {
    double R[9];
    double t[3];
    double C[3];
    double fx, fy, cx, cy;
    int32_t width, height;
} isg_camera;

/* Pre-activation Gaussian parameters (gaussians.py:27-78), row-major per
 * parameter: positions (n,3), log_scales (n,3), rotations (n,4) wxyz,
 * opacity_logits (n), sh (n,K,3) with K = (degree+1)^2.  dtype: ISG_F32/F64. */
typedef struct isg_params {
    const void *positions;
    const void *log_scales;
    const void *rotations;
    const void *opacity_logits;
    const void *sh;
    int64_t n;
    int32_t degree;
    int32_t dtype;
} isg_params;

/* Outputs of isg_preprocess, all indexed by cloud row i (length n).
 * key[i]  : depth bits (fp64, ascending as uint64) if visible, else ~0.
 * rect[i] : inclusive tile rect (tx0, ty0, tx1, ty1), int32 x4.
 * feat    : raster features, 12 values of feat_dtype per row:
 *           (mx, my, conic_a, conic_b, conic_c, opacity, r, g, b, 0, 0, 0).
 * flag[i] : 1 if kept (rasterizer.py:142-158 `keep`).
 * full64  : optional (NULL to skip) reference SplatBatch columns in float64,
 *           16 per row: mean2d(2) cov2d(3) conic(3) depth color(3) opacity
 *           pad(3). */
typedef struct isg_preprocess_out {
    uint64_t *key;
    int32_t *rect;
    void *feat;
    uint8_t *flag;
    double *full64;
    int32_t feat_dtype;
} isg_preprocess_out;

/* Replaces _project_kernel (_kernels.py:144-198) + the keep mask of
 * project (rasterizer.py:105-158). fp64 arithmetic, no FMA contraction,
 * glibc-exact exp: depth/mean2d/cov2d/conic/rect are bit-exact. */
int isg_preprocess(const isg_params *p, const isg_camera *cam, int32_t tile_size,
                   const isg_preprocess_out *out, void *stream);

/* isg_preprocess with the camera in DEVICE memory (an isg_camera the caller
 * uploads before the launch), float32 parameters and features: a launch that
 * can be captured into a CUDA graph and replayed for every view. */
int isg_preprocess_devcam(const isg_params *p, const isg_camera *cam_dev, int32_t width,
                          int32_t height, int32_t tile_size, const isg_preprocess_out *out,
                          void *stream);

/* Stable radix sort of (uint64 key, int32 value) pairs over key bits
 * [begin_bit, end_bit).  Replaces np.lexsort((indices, depth))
 * (rasterizer.py:161-163, engine.py:214) when values are in index order.
 * Call with workspace == NULL to get *ws_bytes. */
int isg_sort_u64(void *workspace, size_t *ws_bytes, const uint64_t *keys_in,
                 uint64_t *keys_out, const int32_t *vals_in, int32_t *vals_out,
                 int64_t n, int32_t begin_bit, int32_t end_bit, void *stream);

/* Same for (uint32 key, int32 value) pairs (tile binning). */
/* The depth order (np.lexsort((indices, depth)), rasterizer.py:161-163):
 * stable sort of (float64 depth bits, id) pairs, bit-identical to
 * isg_sort_u64 over bits [0, 64) but with 5 radix passes (top 40 bits) and a
 * fix-up of equal-top-40 runs.  Workspace as isg_sort_u64. */
int isg_sort_depth(void *workspace, size_t *ws_bytes, const uint64_t *keys_in,
                   uint64_t *keys_out, const int32_t *vals_in, int32_t *vals_out, int64_t n,
                   void *stream);

int isg_sort_u32(void *workspace, size_t *ws_bytes, const uint32_t *keys_in,
                 uint32_t *keys_out, const int32_t *vals_in, int32_t *vals_out,
                 int64_t n, int32_t begin_bit, int32_t end_bit, void *stream);

/* Binning, stage 1 (_count_tile_entries, _kernels.py:202-211 + the cumsum of
 * rasterizer.py:183-184): gather per-rank rect/features into rank order and
 * scan the tile counts of each rect clipped to tile rows [row_lo, row_hi)
 * (the caller's own tiles; all rows for one GPU).  order[r] = row of rank r
 * (the sorted values); ranks whose sorted key is ~0 are culled (0 tiles).
 * emit_off has n+1 entries (exclusive scan); counts[0] = visible ranks M,
 * counts[1] = total entries E (int64, device).  Workspace as above.
 * isg_bin_count_rows: the same over the 64-byte payload rows of received
 * splat records (rect, 12 float32 features; isg_route_pack), float32. */
int isg_bin_count_rows(void *workspace, size_t *ws_bytes, int64_t n, const uint64_t *sorted_keys,
                       const int32_t *order, const int32_t *payload, int32_t row_lo,
                       int32_t row_hi, int32_t *rect_sorted, float *feat_sorted, int64_t *emit_off,
                       int64_t *counts, void *stream);
int isg_bin_count(void *workspace, size_t *ws_bytes, int64_t n, const uint64_t *sorted_keys,
                  const int32_t *order, const int32_t *rect, const void *feat,
                  int32_t feat_dtype, int32_t row_lo, int32_t row_hi, int32_t *rect_sorted,
                  void *feat_sorted, int64_t *emit_off, int64_t *counts, void *stream);

/* Row -> rank inverse of the depth order: rank_of[order[r]] = r for
 * visible ranks (sorted key != ~0), -1 for culled rows.  n <= INT32_MAX. */
int isg_rank_of(int64_t n, const uint64_t *sorted_keys, const int32_t *order, int32_t *rank_of,
                void *stream);

/* Binning, stage 2 (_fill_tile_entries, _kernels.py:215-225): emit
 * (tile id - row_lo*tiles_x, rank) pairs in rank order for ranks [0, m),
 * rects clipped to tile rows [row_lo, row_hi) exactly as in isg_bin_count. */
int isg_bin_emit(int64_t m, const int32_t *rect_sorted, const int64_t *emit_off,
                 int32_t tiles_x, int32_t row_lo, int32_t row_hi, uint32_t *tile_keys,
                 int32_t *tile_vals, void *stream);


/* 16-bit tile-key variants (band of at most 65536 tiles, e.g. 4096^2 at
 * 16 px): the same pairs / order / offsets as isg_bin_emit + isg_sort_u32 +
 * isg_tile_offsets, with 2-byte keys (25 % less traffic in the tile sort). */
int isg_bin_emit16(int64_t m, const int32_t *rect_sorted, const int64_t *emit_off,
                   int32_t tiles_x, int32_t row_lo, int32_t row_hi, uint16_t *tile_keys,
                   int32_t *tile_vals, void *stream);
int isg_sort_u16(void *workspace, size_t *ws_bytes, const uint16_t *keys_in, uint16_t *keys_out,
                 const int32_t *vals_in, int32_t *vals_out, int64_t n, int32_t begin_bit,
                 int32_t end_bit, void *stream);
int isg_tile_offsets16(int64_t e, const uint16_t *sorted_tile_keys, int32_t n_tiles,
                       int32_t *offsets, void *stream);

/* Binning, stage 3: CSR tile offsets from sorted tile keys (n_tiles+1). */
int isg_tile_offsets(int64_t e, const uint32_t *sorted_tile_keys, int32_t n_tiles,
                     int32_t *offsets, void *stream);

/* Forward composite (_forward_tiles, _kernels.py:229-278) over the tile rows
 * [row_lo, row_hi) of a tiles_x-wide grid; offsets (CSR, relative to
 * row_lo*tiles_x) and entries (ranks) come from binning.  If tile_ids is
 * non-NULL the CTAs instead walk the n_tiles listed tile ids (the
 * reference's arbitrary `own_tiles`) with offsets indexed by list slot.
 * Outputs (full-image, row-major): image (H,W,3) in image_dtype, t_final
 * (H,W) in feat_dtype, n_last (H,W) = 1 + index (within the tile's list) of
 * the last composited entry, n_contrib (H,W) optional, n_iter (H,W) optional
 * (entries iterated before the stop: the reference's loop trip count, for
 * the roofline's pair counts), touched (per rank, int64) optional.
 * bg: 3 doubles (host values). */
int isg_raster_fwd(int32_t feat_dtype, int32_t width, int32_t height, int32_t tiles_x,
                   int32_t row_lo, int32_t row_hi, const int32_t *tile_ids, int32_t n_tile_ids,
                   const int32_t *offsets,
                   const int32_t *entries, const void *feat_sorted, const double *bg,
                   void *image, int32_t image_dtype, void *t_final, int32_t *n_last,
                   int32_t *n_contrib, int32_t *n_iter, int64_t *touched, void *stream);

/* L1 + D-SSIM loss and its exact image gradient (metrics.py:135-189) over
 * full images (H,W,3) of `dtype`.  ref is `dtype`, or 8-bit codes k when
 * ref_u8 != 0 (read as float(k / 255.0), exactly the reference's PNG load).
 * grad gets dL/dimage in `dtype`; the loss scalar (float64) lands in
 * *loss_dev.  Workspace as above. */
int isg_loss_l1_dssim(void *workspace, size_t *ws_bytes, int32_t dtype, int32_t height,
                      int32_t width, const void *image, const void *ref, int32_t ref_u8,
                      double lambda_dssim, void *grad, double *loss_dev, void *stream);

/* Block-partial array sizes of the loss (16x16 centre / pixel blocks over
 * the full image). */
int isg_loss_partials_size(int32_t height, int32_t width, int32_t *n_ssim, int32_t *n_l1);

/* Loss and gradient for the pixel rows [row0, row1) of a band (row0 a
 * multiple of 16; row1 a multiple of 16 or H).  image points at global row
 * img_row0 and must cover rows [row0-16, row1+10) clipped to [0, H); ref is
 * the full (H,W,3) ground truth.  grad receives rows [row0, row1) (pointer at
 * row0).  The band's own 16x16 block partials are written into the
 * full-image arrays part_ssim / part_l1 (other entries untouched), so
 * summing the bands' arrays and calling isg_loss_finish gives exactly the
 * single-band loss. */
int isg_loss_rows(void *workspace, size_t *ws_bytes, int32_t dtype, int32_t height,
                  int32_t width, int32_t row0, int32_t row1, const void *image, int32_t img_row0,
                  const void *ref, int32_t ref_u8, double lambda_dssim, void *grad,
                  double *part_ssim, double *part_l1, void *stream);

/* Fixed-order final sum of the block partials into *loss_dev. */
int isg_loss_finish(int32_t height, int32_t width, double lambda_dssim, const double *part_ssim,
                    const double *part_l1, double *loss_dev, void *stream);

/* Mean SSIM over valid centres (metrics.py:105-132) of (H,W,C) float64
 * images, into *out_dev. */
int isg_ssim(void *workspace, size_t *ws_bytes, int32_t height, int32_t width,
             int32_t channels, const double *image, const double *ref, double *out_dev,
             void *stream);

/* Per-tile backward (_backward_tiles, _kernels.py:282-374).  Writes the
 * per-(tile, splat) subtotals as 9 values (dmean 2, dconic 3, dcolor 3,
 * dopac 1, feat_dtype; float32 records are padded to a 12-float / 48-byte
 * stride, float64 records are 9 doubles) into slot emit_off[rank] + (index of the tile inside
 * the rank's row-clipped rect), i.e. splat-major with tiles ascending --
 * exactly the order in which _reduce_scratch folds them.  With emit_off ==
 * NULL the subtotal of entry e goes to slot e instead (the reference's
 * scratch layout, rasterizer.py:218-245).  tile_ids as in isg_raster_fwd. */
int isg_raster_bwd(int32_t feat_dtype, int32_t width, int32_t height, int32_t tiles_x,
                   int32_t row_lo, int32_t row_hi, const int32_t *tile_ids, int32_t n_tile_ids,
                   const int32_t *offsets,
                   const int32_t *entries, const void *feat_sorted, const int32_t *rect_sorted,
                   const int64_t *emit_off, const double *bg, const void *t_final,
                   const int32_t *n_last, const void *dl_dimage, int32_t dl_dtype,
                   void *partials, void *stream);

/* float32 raster pair with contribution masks: the forward also writes, per
 * (tile, 8x8 quadrant, batch of 32 consecutive list entries), a 32-bit mask
 * of the entries some pixel of the quadrant composited; the backward given
 * the same array stages only those entries (the others have all-zero
 * subtotals, written as zeros).  Results equal isg_raster_fwd / isg_raster_bwd
 * with feat_dtype ISG_F32.  contrib_mask holds isg_contrib_mask_words(E,
 * n_tiles) uint32 words for a launch over n_tiles tiles with E list entries;
 * it needs no initialisation.  The two calls must see the same tiles,
 * offsets and n_last.  slot_rank (optional): the lists are live-only
 * subtotal slots (isg_bin_emit_live); entries map to ranks through it and the
 * backward writes each list entry's record at that slot with its tile row as
 * int32 bits in float 9.  tile_order (optional, n_tiles entries): CTA b
 * processes list position tile_order[b] -- the launch order only (heaviest
 * lists first, isg_tile_order); results do not depend on it. */
int64_t isg_contrib_mask_words(int64_t n_entries, int32_t n_tiles);

/* Backward list chunking (optional argument of the masked raster pair): the
 * backward runs each tile's list as chunks of `chunk` entries (a multiple of
 * 32), each its own CTA, so a long list no longer serialises the end of the
 * launch.  The forward leaves, per pixel, (T, r, g, b) before every internal
 * chunk boundary in `state` (isg_chunk_state_floats floats); the backward
 * starts a chunk from that state (S = image - accumulated colour).  `items`
 * / `n_items` come from isg_chunk_items (max_items = isg_chunk_items_max).
 * The chunk size must not depend on the partition (bitwise W-invariance). */
typedef struct isg_chunks {
    int32_t chunk;          /* entries per backward work item; 0 = one item per tile */
    float *state;           /* forward -> backward state at chunk boundaries */
    const int32_t *items;   /* (tile list position, chunk) int32 pairs */
    const int32_t *n_items; /* device count of items */
    int32_t max_items;      /* grid of the backward launch */
    const float *image;     /* the forward's float32 image (same pixels as t_final) */
    int32_t *tile_last;     /* forward -> items: last composited position per (tile, quadrant), 4 x n_tiles */
    int32_t unroll2;        /* unchunked backward: several entries per step (same results; for
                               launches of about one wave, whose tails run one warp per SM) */
} isg_chunks;
int64_t isg_chunk_state_floats(int64_t n_entries, int32_t n_tiles, int32_t chunk);
int32_t isg_chunk_items_max(int64_t n_entries, int32_t n_tiles, int32_t chunk);
/* Work items in launch order, built between the forward and the backward:
 * for every list position of tile_order (NULL: 0..n_tiles-1) with tile_last
 * maximum L over its quadrants, split != 0: ceil(L / chunk) chunks (at least
 * one; the last one runs to the end of the list, whose entries past L
 * contribute nothing); split == 0: one item for the whole list.  Written as
 * (position, chunk | 1 << 30 for the last) pairs; *n_items (device) = their
 * number.  A chunk restart rounds differently from an unbroken walk, so the
 * chunking is part of the arithmetic (engine.py: it follows the image). */
int isg_chunk_items(int32_t n_tiles, const int32_t *offsets, const int32_t *tile_order,
                    const int32_t *tile_last, int32_t chunk, int32_t split, int32_t *items,
                    int32_t *n_items, void *stream);
int isg_raster_fwd_masked(int32_t width, int32_t height, int32_t tiles_x, int32_t row_lo,
                          int32_t row_hi, const int32_t *tile_ids, int32_t n_tile_ids,
                          const int32_t *tile_order, const int32_t *offsets, const int32_t *entries, const void *feat_sorted,
                          const double *bg, void *image, int32_t image_dtype, void *t_final,
                          int32_t *n_last, int32_t *n_contrib, int32_t *n_iter, int64_t *touched,
                          uint32_t *contrib_mask, const isg_chunks *chunks,
                          const int32_t *slot_rank, void *stream);
int isg_raster_bwd_masked(int32_t width, int32_t height, int32_t tiles_x, int32_t row_lo,
                          int32_t row_hi, const int32_t *tile_ids, int32_t n_tile_ids,
                          const int32_t *tile_order, const int32_t *offsets, const int32_t *entries, const void *feat_sorted,
                          const int32_t *rect_sorted, const int64_t *emit_off, const double *bg,
                          const void *t_final, const int32_t *n_last, const void *dl_dimage,
                          int32_t dl_dtype, void *partials, const uint32_t *contrib_mask,
                          const isg_chunks *chunks, const int32_t *slot_rank, void *stream);

/* The sort and the CSR offsets with the item count on the device (*n_dev,
 * *e_dev; n_max / e_max host-side upper bounds that size grids and the
 * workspace): the band path sorts its live-only lists without a host sync.
 * key_bytes 2, 4 or 8. */
int isg_sort_pairs_dev(void *workspace, size_t *ws_bytes, int32_t key_bytes, const void *keys_in,
                       void *keys_out, const int32_t *vals_in, int32_t *vals_out, int64_t n_max,
                       const int64_t *n_dev, int32_t begin_bit, int32_t end_bit, void *stream);
int isg_tile_offsets_dev(int64_t e_max, const int64_t *e_dev, const void *sorted_keys,
                         int32_t key_bytes, int32_t n_tiles, int32_t *offsets, void *stream);

/* Heaviest-first launch order in one launch: tiles bucketed by the bit length
 * of their list, longest buckets first (order inside a bucket arbitrary; the
 * raster results do not depend on the launch order). */
int isg_tile_order(int32_t n_tiles, const int32_t *offsets, int32_t *order, void *stream);

/* Heaviest-first launch order of n_tiles tile lists: keys16[t] = 65535 -
 * min(list length, 65535) and vals[t] = t, to be sorted ascending with
 * isg_sort_u16 (16 bits) into the tile_order of the raster pair.
 * heavy_pct > 0: only lists of at least heavy_pct % of the mean length go
 * first (by length); the rest follow in list order (spatial locality). */
int isg_tile_order_keys(int32_t n_tiles, const int32_t *offsets, int32_t heavy_pct,
                        uint16_t *keys16, int32_t *vals, void *stream);

/* The ordered fold over the live-only layout (float32 records of
 * isg_raster_bwd_masked with slot_rank: rank r's slots live_off[r] ..
 * live_off[r + 1], tile row in float 9), canonical blocks of canon_rows >= 1
 * tile rows: bit-identical to isg_reduce_ordered over the full layout (the
 * uncomposited pairs' zero subtotals only ever add zeros). */
int isg_reduce_live(int64_t m, const int64_t *live_off, const float *partials,
                    const int32_t *order, const int32_t *rect_sorted, int32_t row_lo,
                    int32_t row_hi, int32_t canon_rows, double *grad2d, double *grad_norm,
                    void *stream);

/* Live-only binning (the float32 training lists): isg_bin_count plus, per
 * rank, the tiles some pixel can composite (the rasteriser's conservative box
 * test): live_off (n+1, exclusive scan), live_mask (bit k = k-th tile of the
 * clipped rect in row-major order, rects of <= 64 tiles) and counts[2] = live
 * total.  rect/feat (float32 SoA) or payload (64-byte rows).  isg_bin_emit_live
 * then writes the live (tile, slot) pairs compacted in rank order: keys[p] =
 * band tile, slot_rank[p] = rank for slot p in [0, live total) (one thread
 * per rank; emit_off is not read, kept for the call's symmetry with
 * isg_bin_emit). */
int isg_bin_count_live(void *workspace, size_t *ws_bytes, int64_t n, const uint64_t *sorted_keys,
                       const int32_t *order, const int32_t *rect, const int32_t *payload,
                       const float *feat, int32_t row_lo, int32_t row_hi, int32_t *rect_sorted,
                       float *feat_sorted, int64_t *emit_off, int64_t *live_off,
                       uint64_t *live_mask, int64_t *counts, void *stream);

/* The training variant of isg_bin_count_live (float32 SoA rect/feat): no
 * full-layout offsets (emit_off is not produced and counts[1] stays 0: the
 * live lists never read them) and, when rank_of is given, the row -> rank
 * inverse of isg_rank_of in the same pass. */
int isg_bin_count_train(void *workspace, size_t *ws_bytes, int64_t n, const uint64_t *sorted_keys,
                        const int32_t *order, const int32_t *rect, const float *feat,
                        int32_t row_lo, int32_t row_hi, int32_t *rect_sorted, float *feat_sorted,
                        int64_t *live_off, uint64_t *live_mask, int32_t *rank_of, int64_t *counts,
                        void *stream);
int isg_bin_emit_live(int64_t m, const int32_t *rect_sorted, const int64_t *emit_off,
                      const int64_t *live_off, const uint64_t *live_mask, const float *feat_sorted,
                      int32_t tiles_x, int32_t row_lo, int32_t row_hi, void *tile_keys,
                      int32_t key_bytes, int32_t *slot_rank, void *stream);

/* Ordered fold (_reduce_scratch, _kernels.py:398-411): for rank r < m sum its
 * subtotal slots [emit_off[r], emit_off[r+1]) in float64 and write
 * grad2d[order[r]] (9 doubles).  canon_rows <= 0: the reference's single-level
 * fold in ascending tile order.  canon_rows > 0: the canonical two-level fold
 * used by the training step -- tiles ascending inside each block of
 * canon_rows tile rows, then block sums ascending -- whose grouping does not
 * depend on the GPU count (needs rect_sorted and the band rows).  If
 * grad_norm is non-NULL it receives hypot(dmean) at row order[r]
 * (rasterizer.py:397).  order == NULL writes grad2d in rank order (row r =
 * rank r) instead of at row order[r]: coalesced, for consumers indexed
 * through isg_rank_of. */
int isg_reduce_ordered(int32_t feat_dtype, int64_t m, const int64_t *emit_off,
                       const void *partials, const int32_t *order, const int32_t *rect_sorted,
                       int32_t row_lo, int32_t row_hi, int32_t canon_rows, double *grad2d,
                       double *grad_norm, void *stream);

/* ---- multi-GPU data plane (distributed.py:127-226, engine.py:201-237,
 * 499-507), row-band pixel partition.  band_rows / shard_start are HOST
 * arrays of n+1 boundaries (n <= 64). ---- */

/* Exclusive scan of n int64 counts: off[0..n], *total = off[n] (device). */
int isg_scan_i64(void *workspace, size_t *ws_bytes, int64_t n, const int64_t *cnt, int64_t *off,
                 int64_t *total, void *stream);

/* Route plan of a shard: per plan block of 256 rows and per band, the
 * exclusive prefixes of the rows' splat records (1 per band reached) and
 * canonical-block gradient records (blocks of canon_rows tile rows inside the
 * band), plus per-band totals[3 * d + {0, 1, 2}] = (splat records, block
 * records, tile entries).  A visible row reaches the contiguous band range its
 * rect's tile rows overlap (_route_mask, _kernels.py:378-394, for row bands).
 * plan holds isg_route_plan_size() int64 elements. */
int isg_route_plan_size(int64_t n, int32_t n_bands, int64_t *plan_elems);
int isg_route_plan(int64_t n, const uint8_t *flag, const int32_t *rect, const int32_t *band_rows,
                   int32_t n_bands, int32_t canon_rows, int64_t *plan, int64_t *totals,
                   void *stream);

/* Splat records (the reference's mailbox `splats`, engine.py:201-215): for
 * each band d a row reaches, its depth key at keys[dest_off[d] + j] and a
 * 64-byte payload (rect, 12 float32 raster features) at pay[...], j = the
 * row's rank among the shard rows reaching d (shard row order).  Band
 * self_band's records go to keys_self / pay_self (this rank's receive
 * buffers), every other band's to keys_send / pay_send.  dest_off: HOST. */
int isg_route_pack(int64_t n, const uint8_t *flag, const int32_t *rect, const uint64_t *key,
                   const float *feat, const int32_t *band_rows, int32_t n_bands,
                   const int64_t *plan, const int64_t *dest_off, int32_t self_band,
                   uint64_t *keys_send, int32_t *pay_send, uint64_t *keys_self,
                   int32_t *pay_self, void *stream);

/* Render-API glue (rasterizer.py's SplatBatch columns).  isg_compact_count:
 * pos[0..n] = exclusive scan of the keep flags (pos[n] = kept rows, device;
 * two-phase workspace).  isg_compact_batch: each kept row i of
 * isg_preprocess's full64 / rect (indices optional: NULL = row id) to column
 * position pos[i] of mean2d (m,2), cov2d (m,3), conic (m,3), depth, colour
 * (m,3), opacity, tile_min / tile_max (m,2) int32, indices int64 -- the
 * reference's stable `keep` compaction (rasterizer.py:142-158).
 * isg_gather_batch: sorted row r <- column row order[r]: the 12 raster
 * features in feat_dtype and the int32 tile rect (rasterizer.py:294-345). */
int isg_compact_count(void *workspace, size_t *ws_bytes, int64_t n, const uint8_t *flag,
                      int64_t *pos, void *stream);
int isg_compact_batch(int64_t n, const uint8_t *flag, const int64_t *pos, const double *full64,
                      const int32_t *rect, const int64_t *indices, double *mean2d, double *cov2d,
                      double *conic, double *depth, double *color, double *opacity,
                      int32_t *tile_min, int32_t *tile_max, int64_t *indices_out, void *stream);
int isg_gather_batch(int64_t m, const int64_t *order, const double *mean2d, const double *conic,
                     const double *color, const double *opacity, const int32_t *tile_min,
                     const int32_t *tile_max, int32_t feat_dtype, void *feat, int32_t *rect,
                     void *stream);

/* Peer-store variant of isg_route_pack (the fused pack + exchange): band d's
 * records go to keys_dst[d][j] / pay_dst[d][16 * j] (int32 units), j as
 * above -- keys_dst/pay_dst are HOST arrays of n_bands DEVICE pointers, each
 * already offset to where this shard's segment starts in band d's receive
 * buffers.  For d != this rank they point into the peer GPU's memory mapped
 * into this process (NVLink stores; e.g. torch symmetric memory), so the
 * exchange is the pack kernel's own stores.  pay_dst entries 16-byte aligned.
 * Replaces the mailbox put of engine.py:201-215 (the caller adds a barrier
 * before the bands read). */
int isg_route_pack_peer(int64_t n, const uint8_t *flag, const int32_t *rect, const uint64_t *key,
                        const float *feat, const int32_t *band_rows, int32_t n_bands,
                        const int64_t *plan, uint64_t *const *keys_dst, int32_t *const *pay_dst,
                        void *stream);

/* The reference's round-robin routing mask (route_rows, distributed.py:127-136
 * over _route_mask, _kernels.py:378-394): rects (n, 4) int32 (tile_min,
 * tile_max); mask (n, workers) u8, 1 iff the rect touches a tile whose linear
 * id is congruent to w.  workers <= 64. */
int isg_route_mask(int64_t n, const int32_t *rects, int32_t tiles_x, int32_t workers,
                   uint8_t *mask, void *stream);

/* Canonical blocks (canon_rows tile rows) of each received splat's rect
 * inside the band [row_lo, row_hi) (payload rows as isg_route_pack). */
int isg_band_blocks(int64_t r, const int32_t *payload, int32_t row_lo, int32_t row_hi,
                    int32_t canon_rows, int64_t *nb, void *stream);

/* Band fold (the per-tile GradChunks of engine.py:256-284, pre-folded):
 * rank r's float32 subtotals folded per canonical block (float64, tiles
 * ascending) into 9-double records at gbuf[9 * (gpos[order[r]] + b)] --
 * records by receive index, so each source rank's segment is its own rows'
 * records in its shard row order.  live_layout: emit_off is the live-only
 * slot offsets (isg_bin_emit_live; records carry their tile row) and every
 * block of the rank's clipped rows in [row_lo, row_hi) gets a record. */
int isg_band_fold(int64_t m, const int64_t *emit_off, const float *partials,
                  const int32_t *rect_sorted, const int32_t *order, const int64_t *gpos,
                  int32_t row_lo, int32_t row_hi, int32_t canon_rows, int32_t live_layout,
                  double *gbuf, void *stream);

/* Peer-store variant of isg_band_fold (the fused fold + gradient exchange,
 * engine.py:256-284 / 499-507): receive indices [recv_end[s-1], recv_end[s])
 * came from source rank s (recv_end HOST, n_src entries, last >= m), whose
 * records go to dst_base[s] + 9 * gpos[...] -- dst_base a HOST array of
 * DEVICE pointers (the owner's gradient receive buffer, on its GPU, offset so
 * that its gpos range lands at this band's segment). */
int isg_band_fold_peer(int64_t m, const int64_t *emit_off, const float *partials,
                       const int32_t *rect_sorted, const int32_t *order, const int64_t *gpos,
                       int32_t row_lo, int32_t row_hi, int32_t canon_rows, int32_t live_layout,
                       int32_t n_src, const int64_t *recv_end, double *const *dst_base,
                       void *stream);

/* Device-to-device copy of `bytes` on `stream` (either side may be a peer
 * GPU's memory mapped into this process): the halo rows of the peer exchange,
 * which replace the reference's full-canvas `frag` exchange (engine.py:229-237). */
int isg_copy(void *dst, const void *src, int64_t bytes, void *stream);

/* Band raster cost per canonical block (load balance of the row bands):
 * hist[(prow0 + y) / (16 * canon_rows)] += sum_x n_last[y][x] for the band's
 * pixel rows [prow0, prow1) (n_last band-local, width per row), as exact
 * integer sums in float64. */
int isg_band_cost(const int32_t *n_last, int32_t prow0, int32_t prow1, int32_t width,
                  int32_t canon_rows, double *hist, void *stream);

/* Owner fold over the route plan (reduce_gradients_fused,
 * distributed.py:178-226): per shard row, the block records of the bands it
 * reached (seg[d]: HOST array of device pointers to band d's records for
 * this shard) summed bands ascending, blocks ascending, in float64 -- the
 * canonical two-level fold, bit-identical to isg_reduce_ordered with
 * canon_rows.  Rows not visible get zeros. */
int isg_owner_fold_plan(int64_t n, const uint8_t *flag, const int32_t *rect,
                        const int32_t *band_rows, int32_t n_bands, int32_t canon_rows,
                        const int64_t *plan, const double *const *seg, double *grad2d,
                        void *stream);

/* Keys (owner-local rows) and identity values of received gradient records. */
int isg_grad_rows(int64_t r, const int32_t *records, uint32_t *rows, int32_t *idx, void *stream);

/* Owner fold (reduce_gradients_fused, distributed.py:178-226): per shard row
 * the records seg_off[i]..seg_off[i+1] (perm into records, arrival order) are
 * summed in float64 into grad2d[i]; rows without records are left untouched. */
int isg_owner_fold(int64_t n_rows, const int32_t *seg_off, const int32_t *perm,
                   const int32_t *records, double *grad2d, void *stream);

/* 2D -> 3D chain rule (_chain_kernel, _kernels.py:415-634) for rows with
 * flag != 0; grad2d is (n, 9) float64.  Outputs (parameter dtype, same
 * shapes as isg_params) are fully written (zeros for unflagged rows). */
int isg_chain(const isg_params *p, const isg_camera *cam, const uint8_t *flag,
              const double *grad2d, void *d_positions, void *d_log_scales,
              void *d_rotations, void *d_opacity_logits, void *d_sh, void *stream);

/* Dense Adam (optim.py:20-56) over n elements, numpy weak-scalar semantics:
 * constants are given already rounded to the storage dtype. */
typedef struct isg_adam_consts {
    double b1, omb1, b2, omb2, bc1, bc2, lr, eps;
} isg_adam_consts;

int isg_adam(int32_t dtype, int64_t n, void *p, const void *g, void *m, void *v,
             const isg_adam_consts *c, void *stream);

/* Fused training update for float32 parameters: chain rule for flagged rows,
 * TrainStats update (engine.py:508-515) and Adam for all n rows and five
 * groups (engine.py:524-536), one pass.  m/v mirror the parameter layout.
 * lr[5] in PARAM_NAMES order; stats_seen/grad_accum optional. */
typedef struct isg_train_state {
    float *positions, *log_scales, *rotations, *opacity_logits, *sh;
    float *m_positions, *m_log_scales, *m_rotations, *m_opacity_logits, *m_sh;
    float *v_positions, *v_log_scales, *v_rotations, *v_opacity_logits, *v_sh;
    int64_t *seen;
    double *grad_accum;
    int64_t n;
    int32_t degree;
} isg_train_state;

/* densify_and_prune's row classification (training.py:334-347) on the device,
 * float64 with the glibc-exact exp like the reference's numpy: per row cls =
 * 0 keep, 1 clone, 2 split, 3 prune.  log_scales (n, 3) and logits (n)
 * float32; seen int64, grad_accum float64 (TrainStats); scale_prune applies
 * when scale_prune_on. */
int isg_densify_classify(int64_t n, const float *log_scales, const float *logits,
                         const int64_t *seen, const double *grad_accum, double opacity_prune,
                         double scale_prune, int32_t scale_prune_on, double grad_threshold,
                         double split_threshold, uint8_t *cls, void *stream);

int isg_chain_adam(const isg_train_state *s, const isg_camera *cam, const uint8_t *flag,
                   const double *grad2d, const float *lr5, const isg_adam_consts *c,
                   double half_w, double half_h, void *stream);

/* Training-step split of isg_chain_adam: chain rule + TrainStats for float32
 * parameters (grads written for every row, zeros when unflagged) ... */
int isg_chain_train(const isg_params *p, const isg_camera *cam, const uint8_t *flag,
                    const double *grad2d, float *d_positions, float *d_log_scales,
                    float *d_rotations, float *d_opacity_logits, float *d_sh, int64_t *seen,
                    double *grad_accum, double half_w, double half_h, void *stream);

/* isg_chain_train over a rank-ordered grad2d (isg_reduce_ordered with
 * order == NULL): row i reads the 2-D gradients of rank rank_of[i]
 * (isg_rank_of); rows with rank -1 are not visible (zero gradients). */
int isg_chain_train_ranked(const isg_params *p, const isg_camera *cam, const int32_t *rank_of,
                           const double *grad2d_ranked, float *d_positions, float *d_log_scales,
                           float *d_rotations, float *d_opacity_logits, float *d_sh,
                           int64_t *seen, double *grad_accum, double half_w, double half_h,
                           void *stream);

/* The live fold fused into the ranked chain (the training step on live-only
 * lists): row i folds the live subtotal slots of its rank r = rank_of[i]
 * (live_off[r] .. live_off[r+1] of partials; rect_sorted, [row_lo, row_hi),
 * canon_rows as isg_reduce_live -- bit-identical sums) and runs the chain
 * rule on them; grad2d_out (optional) receives the rank-ordered 2-D
 * gradients. */
int isg_chain_fold_train(const isg_params *p, const isg_camera *cam, const int32_t *rank_of,
                         const int64_t *live_off, const float *partials,
                         const int32_t *rect_sorted, int32_t row_lo, int32_t row_hi,
                         int32_t canon_rows, double *grad2d_out, float *d_positions,
                         float *d_log_scales, float *d_rotations, float *d_opacity_logits,
                         float *d_sh, int64_t *seen, double *grad_accum, double half_w,
                         double half_h, void *stream);

/* The whole per-Gaussian tail of a training step in one pass: the live fold
 * and chain rule of isg_chain_fold_train, TrainStats, then the dense Adam
 * update of every row's 23 parameters (isg_adam_groups' arithmetic, bit for
 * bit: engine.py:508-536, optim.py:20-56) without the parameter gradients
 * leaving registers.  grads_out: NULL, or 5 float32 arrays (PARAM_NAMES order)
 * that also receive the gradients; lr5 HOST, PARAM_NAMES order. */
int isg_chain_fold_adam(const isg_train_state *s, const isg_camera *cam, const int32_t *rank_of,
                        const int64_t *live_off, const float *partials, const int32_t *rect_sorted,
                        int32_t row_lo, int32_t row_hi, int32_t canon_rows, double *grad2d_out,
                        float *const *grads_out, const float *lr5, const isg_adam_consts *c,
                        double half_w, double half_h, void *stream);

/* The same single pass from row-ordered 2-D gradients (rows with flag set;
 * the sharded step's owner fold, isg_owner_fold_plan): float32 chain rule +
 * TrainStats + dense Adam, the gradients kept in registers (grads_out
 * optional as above).  The float32 training counterpart of isg_chain_adam. */
int isg_chain_adam_train(const isg_train_state *s, const isg_camera *cam, const uint8_t *flag,
                         const double *grad2d, float *const *grads_out, const float *lr5,
                         const isg_adam_consts *c, double half_w, double half_h, void *stream);

/* ... then dense float32 Adam over up to 8 groups in one launch (arrays of
 * `count` host-side pointers / sizes / learning rates; constants as for
 * isg_adam).  Bit-identical to isg_adam per element. */
int isg_adam_groups(int32_t count, float *const *p, const float *const *g, float *const *m,
                    float *const *v, const int64_t *n, const float *lr, const isg_adam_consts *c,
                    void *stream);

/* glibc-exact exp over an array (verification hook for the key path). */
int isg_exp_f64(int64_t n, const double *x, double *y, void *stream);

/* FP32 FMA-pipe throughput probe (the measured roofline denominator of the
 * raster kernels): `blocks` x 256 threads, each running 8 independent
 * fma.rn.f32 chains for iters x 16 steps (blocks * 256 * iters * 256 flops).
 * `out` (blocks floats) is never written in practice.  Not a reference
 * interface: measurement support for bench.py. */
int isg_probe_ffma(int32_t blocks, int32_t iters, float *out, void *stream);

/* Library identification: returns a static string (arch, build flags). */
const char *isg_version(void);

/* Exact mean distance to the k (<= 8) nearest neighbours of every point
 * over the reference's bucket grid (_mean_knn_distance_grid,
 * gaussians.py:143-162; _knn_mean_grid, _kernels.py:636-708): points (n,3)
 * float64 row-major; lo (3 host doubles), cell and the grid dims gx, gy, gz
 * as the reference computes them on the host.  Bit-exact.  Two-phase
 * workspace (workspace == NULL: size query). */
int isg_knn_mean_grid(void *workspace, size_t *ws_bytes, const double *points, int64_t n,
                      int32_t k, const double *lo, double cell, int64_t gx, int64_t gy,
                      int64_t gz, double *out, void *stream);

/* ---- dataset generation (next row of SURVEY 8f: volume.py, raycast.py) ----
 * Volumes are float64 (nz, ny, nx) x-fastest on the device; dims = (nx, ny,
 * nz), spacing and origin are 3 HOST values each (VolumeGrid, volume.py:25-62).
 * float64, reference statement order, no FMA contraction: bit-identical. */

/* raycast_isosurface (raycast.py:99-262): first-hit march at `step`, bisection
 * refine, headlight Lambertian shading.  image (H,W,3) float64 and/or codes
 * (H,W,3) uint8 = quantize8 (images.py:9-16); either may be NULL.  albedo and
 * background are 3 host doubles. */
int isg_raycast(const double *data, const int32_t *dims, const double *spacing,
                const double *origin, double isovalue, const isg_camera *cam, double step,
                int32_t refine_steps, const double *albedo, const double *background,
                double *image, uint8_t *codes, void *stream);

/* _axis_crossings (volume.py:197-226), step 1: linear indices (C order over
 * edge starts of the strided sub-lattice) of the edges along data axis
 * axis_data (2 = x, 1 = y, 0 = z) whose ends straddle isovalue; *count
 * (device) receives their number.  idx_out must hold every edge of the axis.
 * Two-phase workspace. */
int isg_iso_edges(void *workspace, size_t *ws_bytes, const double *data, const int32_t *dims,
                  int32_t stride, int32_t axis_data, double isovalue, int64_t *idx_out,
                  int64_t *count, void *stream);

/* Step 2: the crossing points (n,3) float64 of n selected edges. */
int isg_iso_edge_points(const double *data, const int32_t *dims, const double *spacing,
                        const double *origin, int32_t stride, int32_t axis_data,
                        double isovalue, int64_t n, const int64_t *idx, double *positions,
                        void *stream);

/* Unit normals (gradient_central + normalisation, volume.py:146-174,
 * 270-275) at n points (n,3) float64. */
int isg_iso_normals(const double *data, const int32_t *dims, const double *spacing,
                    const double *origin, int64_t n, const double *positions, double *normals,
                    void *stream);

#ifdef __cplusplus
}
#endif
#endif /* ISOGS_H */
