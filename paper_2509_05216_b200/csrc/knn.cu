// knn.cu -- exact k-nearest-neighbour mean distance over a bucket grid
// (init_from_points' scale seeding; gaussians.py:124-162, _kernels.py:636-708).
//
// The host computes the grid exactly as the reference does with numpy (lo,
// cell = 2 cbrt(V / n), dims); the device buckets the points (cell id per
// point, stable radix sort by cell id -> the reference's stable argsort, CSR
// starts by binary search) and one thread per point runs the reference's ring
// search statement for statement: rings of cells at Chebyshev distance `ring`
// expand until the k-th squared distance is <= (ring * cell)^2, the k best
// squared distances are kept sorted by insertion, and the mean of their square
// roots is accumulated in ascending order.  Compiled with -fmad=false (numba
// does not contract), so distances, and therefore the result, are bit-exact.
#include <cub/cub.cuh>

#include "common.cuh"

namespace isg {

constexpr int KNN_MAX_K = 8;

__global__ void __launch_bounds__(256) knn_cell_kernel(int64_t n, const double *__restrict__ pts,
                                                       double lo0, double lo1, double lo2,
                                                       double cell, int64_t gx, int64_t gy,
                                                       int64_t *__restrict__ cell_of,
                                                       int32_t *__restrict__ idx) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    // coords = floor((points - lo) / cell).astype(int64)
    const int64_t cx = (int64_t)floor((pts[3 * i] - lo0) / cell);
    const int64_t cy = (int64_t)floor((pts[3 * i + 1] - lo1) / cell);
    const int64_t cz = (int64_t)floor((pts[3 * i + 2] - lo2) / cell);
    cell_of[i] = (cz * gy + cy) * gx + cx;
    idx[i] = (int32_t)i;
}

__global__ void __launch_bounds__(256) knn_starts_kernel(int64_t n, int64_t n_cells,
                                                         const int64_t *__restrict__ sorted_cells,
                                                         int64_t *__restrict__ starts) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c > n_cells) return;
    int64_t lo = 0, hi = n;  // lower_bound(sorted_cells, c)
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (sorted_cells[mid] < c) lo = mid + 1;
        else hi = mid;
    }
    starts[c] = lo;
}

__global__ void __launch_bounds__(128) knn_mean_kernel(
    int64_t n, const double *__restrict__ pts, const int64_t *__restrict__ cell_of,
    const int32_t *__restrict__ order, const int64_t *__restrict__ starts, int64_t gx, int64_t gy,
    int64_t gz, double cell, int k, double *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double best[KNN_MAX_K];
    const int64_t cid = cell_of[i];
    const int64_t cx = cid % gx, cy = (cid / gx) % gy, cz = cid / (gx * gy);
    const double px = pts[3 * i], py = pts[3 * i + 1], pz = pts[3 * i + 2];
    int found = 0;
    int64_t ring = 0;
    const int64_t max_ring = max(gx, max(gy, gz));
    while (true) {
        const int64_t a0 = max(cx - ring, (int64_t)0), a1 = min(cx + ring, gx - 1);
        const int64_t b0 = max(cy - ring, (int64_t)0), b1 = min(cy + ring, gy - 1);
        const int64_t c0 = max(cz - ring, (int64_t)0), c1 = min(cz + ring, gz - 1);
        for (int64_t c = c0; c <= c1; c++)
            for (int64_t b = b0; b <= b1; b++)
                for (int64_t a = a0; a <= a1; a++) {
                    const int64_t da = cx > a ? cx - a : a - cx;
                    const int64_t db = cy > b ? cy - b : b - cy;
                    const int64_t dc = cz > c ? cz - c : c - cz;
                    if (max(da, max(db, dc)) != ring) continue;
                    const int64_t lin = (c * gy + b) * gx + a;
                    for (int64_t s = starts[lin]; s < starts[lin + 1]; s++) {
                        const int64_t j = order[s];
                        if (j == i) continue;
                        const double dx = pts[3 * j] - px, dy = pts[3 * j + 1] - py,
                                     dz = pts[3 * j + 2] - pz;
                        const double d2 = dx * dx + dy * dy + dz * dz;
                        if (found < k) {
                            best[found++] = d2;
                            if (found == k) {
                                for (int u = 1; u < k; u++) {
                                    const double key = best[u];
                                    int t = u - 1;
                                    while (t >= 0 && best[t] > key) {
                                        best[t + 1] = best[t];
                                        t--;
                                    }
                                    best[t + 1] = key;
                                }
                            }
                        } else if (d2 < best[k - 1]) {
                            int t = k - 2;
                            while (t >= 0 && best[t] > d2) {
                                best[t + 1] = best[t];
                                t--;
                            }
                            best[t + 1] = d2;
                        }
                    }
                }
        const double reach = (double)ring * cell;
        if (found >= k && best[k - 1] <= reach * reach) break;
        if (ring > max_ring) break;
        ring++;
    }
    double acc = 0.0;
    for (int u = 0; u < found; u++) acc += sqrt(best[u]);
    out[i] = acc / (double)max(found, 1);
}

inline size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace isg

using namespace isg;

extern "C" int isg_knn_mean_grid(void *workspace, size_t *ws_bytes, const double *points,
                                 int64_t n, int32_t k, const double *lo, double cell, int64_t gx,
                                 int64_t gy, int64_t gz, double *out, void *stream) {
    if (!ws_bytes || n < 0 || n > INT32_MAX || k < 1 || k > KNN_MAX_K || gx < 1 || gy < 1 ||
        gz < 1 || !(cell > 0.0))
        return (int)cudaErrorInvalidValue;
    const int64_t n_cells = gx * gy * gz;
    size_t sort_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const int64_t *)nullptr,
                                    (int64_t *)nullptr, (const int32_t *)nullptr,
                                    (int32_t *)nullptr, (int)n, 0, 64);
    const size_t need = al256(8 * (size_t)n) * 2 + al256(4 * (size_t)n) * 2 +
                        al256(8 * (size_t)(n_cells + 1)) + al256(sort_bytes);
    if (!workspace) {
        *ws_bytes = need;
        return 0;
    }
    if (*ws_bytes < need || !points || !lo || !out) return (int)cudaErrorInvalidValue;
    if (n == 0) return 0;
    char *w = (char *)workspace;
    int64_t *cell_of = (int64_t *)w;
    w += al256(8 * (size_t)n);
    int64_t *cell_sorted = (int64_t *)w;
    w += al256(8 * (size_t)n);
    int32_t *idx = (int32_t *)w;
    w += al256(4 * (size_t)n);
    int32_t *order = (int32_t *)w;
    w += al256(4 * (size_t)n);
    int64_t *starts = (int64_t *)w;
    w += al256(8 * (size_t)(n_cells + 1));
    cudaStream_t s = (cudaStream_t)stream;
    knn_cell_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, points, lo[0], lo[1], lo[2], cell, gx,
                                                       gy, cell_of, idx);
    ISG_CHECK_LAUNCH();
    // stable by cell id over ascending point index == np.argsort(kind="stable")
    cudaError_t e = cub::DeviceRadixSort::SortPairs(w, sort_bytes, cell_of, cell_sorted, idx,
                                                    order, (int)n, 0, 64, s);
    if (e != cudaSuccess) return (int)e;
    knn_starts_kernel<<<blocks_for(n_cells + 1, 256), 256, 0, s>>>(n, n_cells, cell_sorted,
                                                                   starts);
    ISG_CHECK_LAUNCH();
    knn_mean_kernel<<<blocks_for(n, 128), 128, 0, s>>>(n, points, cell_of, order, starts, gx, gy,
                                                       gz, cell, k, out);
    ISG_CHECK_LAUNCH();
    return 0;
}
