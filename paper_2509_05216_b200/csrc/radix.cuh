// radix.cuh -- the hand-written stable radix sort and exclusive scans
// (radix.cu) used by the binning and data-plane kernels.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace isg {
namespace radix {
// Stable sort of (key, int32 value) pairs on key bits [b0, b1), LSD 8-bit
// digits.  Two-phase workspace (ws == NULL: size query into *ws_bytes).
// keys_in / vals_in are not modified.  n_dev (optional): the item count on
// the device, n its host-side upper bound (grids and workspace from n).
template <typename K>
int sort_pairs(void *ws, size_t *ws_bytes, const K *keys_in, K *keys_out,
               const int32_t *vals_in, int32_t *vals_out, int64_t n, int b0, int b1,
               cudaStream_t s, const int64_t *n_dev = nullptr);
}  // namespace radix

// Exclusive scan of n int64 counts into off[0..n] (off[0] = 0); *total
// (device, optional) = off[n].  Workspace of scan_i64_ws_bytes(n) bytes.
size_t scan_i64_ws_bytes(int64_t n);
int scan_i64(void *ws, size_t ws_bytes, int64_t n, const int64_t *cnt, int64_t *off,
             int64_t *total, cudaStream_t s);
}  // namespace isg
