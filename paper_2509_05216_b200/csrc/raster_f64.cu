// raster_f64.cu -- float64 cross-check rasteriser, the ordered fold and the
// raster C ABI (sm_100a).  The float32 production kernels live in
// raster_f32.cu; this file keeps the reference-exact float64 instantiation.
//
// One CTA per 16x16 tile, one pixel per thread.  Each CTA walks its tile's
// entry list (global compositing order) in batches staged through shared
// memory.  Two instantiations:
//   float  -- production.  The per-pair Gaussian weight uses the SFU
//             (__expf) behind an exact per-splat log threshold so pairs that
//             cannot reach alpha >= 1/255 never touch the SFU; every decision
//             (skip / clamp / stop) is computed by the same inline code in the
//             forward and the backward kernel, so both see identical
//             contributor sets.
//   double -- cross-check build: the reference's arithmetic statement by
//             statement (no FMA contraction: this TU is built with
//             -fmad=false; explicit __fmaf_rn keeps FMAs in the float path)
//             and the glibc-exact exp, so the composite is bit-identical to
//             _forward_tiles (_kernels.py:229-278).
// The backward (_kernels.py:282-374) walks each pixel's contributors back to
// front, recovering T by division from the forward's T_final, reduces the 9
// per-pixel gradient terms of every entry over the CTA (warp shuffles, then
// a fixed-order sum over the 8 warps) and writes one deterministic subtotal
// per (tile, splat) -- the reference's scratch row -- into a splat-major slot
// so the per-splat fold below reads them in ascending tile order.
#include "common.cuh"
#include <type_traits>

#include "fold.cuh"
#include "raster_f32.cuh"

namespace isg {

constexpr int THREADS = 256;
constexpr int FWD_BATCH = 256;
constexpr int BWD_BATCH = 32;
constexpr int WARPS = THREADS / 32;

template <typename T>
struct SplatF {
    T mx, my, a, b, c, op, r, g, bl;
};

__device__ __forceinline__ SplatF<float> load_splat(const float *feat, int rank) {
    const float4 *f = reinterpret_cast<const float4 *>(feat) + 3 * (int64_t)rank;
    float4 x = __ldg(f), y = __ldg(f + 1), z = __ldg(f + 2);
    return SplatF<float>{x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w, z.x};
}

__device__ __forceinline__ SplatF<double> load_splat(const double *feat, int rank) {
    const double2 *f = reinterpret_cast<const double2 *>(feat) + 6 * (int64_t)rank;
    double2 a = __ldg(f), b = __ldg(f + 1), c = __ldg(f + 2), d = __ldg(f + 3), e = __ldg(f + 4);
    return SplatF<double>{a.x, a.y, b.x, b.y, c.x, c.y, d.x, d.y, e.x};
}

// ----------------------------------------------------------- pair kernel ----
// Outcome of one (pixel, splat) pair: 0 = skipped, 1 = composited, 2 = stop.
struct PairF {
    float power, g, alpha;
};

// Float path.  thr = -log(255 o) - 1e-3: below it o*exp(power) < 1/255 holds
// with a margin far above the __expf error, so the skip is exact.
__device__ __forceinline__ bool pair_eval(float px, float py, float mx, float my, float a,
                                          float b, float c, float op, float thr, float &d0,
                                          float &d1, float &g, float &alpha) {
    d0 = px - mx;
    d1 = py - my;
    // power = -0.5 (a d0^2 + c d1^2) - b d0 d1 (exactly rescaled coefficients)
    const float na = -0.5f * a, nb = -b, nc = -0.5f * c;
    const float power = __fmaf_rn(d0, __fmaf_rn(na, d0, __fmul_rn(nb, d1)),
                                  __fmul_rn(__fmul_rn(nc, d1), d1));
    if (power > 0.0f || power < thr) return false;
    g = __expf(power);
    alpha = __fmul_rn(op, g);
    if (alpha > 0.99f) alpha = 0.99f;
    return alpha >= (1.0f / 255.0f);
}

// Double path: _kernels.py:244-262 verbatim.
__device__ __forceinline__ bool pair_eval(double px, double py, double mx, double my, double a,
                                          double b, double c, double op, double /*thr*/,
                                          double &d0, double &d1, double &g, double &alpha) {
    d0 = px - mx;
    d1 = py - my;
    const double power = (-0.5 * (a * d0 * d0 + c * d1 * d1) - b * d0 * d1);
    if (power > 0.0) return false;
    g = exp_glibc(power);
    alpha = op * g;
    if (alpha > ALPHA_CLAMP) alpha = ALPHA_CLAMP;
    return !(alpha < 1.0 / 255.0);
}

__device__ __forceinline__ float skip_threshold(float op) {
    return op > 0.0f ? -__logf(255.0f * op) - 1e-3f : 1.0f;
}
__device__ __forceinline__ double skip_threshold(double) { return 0.0; }

// --------------------------------------------------------------- forward ----
template <typename T, bool TOUCH>
__global__ void __launch_bounds__(THREADS) raster_fwd_kernel(
    int W, int H, int tiles_x, int row_lo, const int32_t *__restrict__ tile_ids,
    const int32_t *__restrict__ offsets, const int32_t *__restrict__ entries,
    const T *__restrict__ feat, T bg0, T bg1, T bg2, void *image, int image_f64,
    T *__restrict__ t_final, int32_t *__restrict__ n_last,
    int32_t *__restrict__ n_contrib, int32_t *__restrict__ n_iter,
    int64_t *__restrict__ touched) {
    __shared__ T s_mx[FWD_BATCH], s_my[FWD_BATCH], s_a[FWD_BATCH], s_b[FWD_BATCH],
        s_c[FWD_BATCH], s_op[FWD_BATCH], s_thr[FWD_BATCH], s_r[FWD_BATCH], s_g[FWD_BATCH],
        s_bl[FWD_BATCH];
    __shared__ int s_rank[TOUCH ? FWD_BATCH : 1];
    const int tl = blockIdx.x;
    const int tid = tile_ids ? tile_ids[tl] : row_lo * tiles_x + tl;
    const int ty = tid / tiles_x, tx = tid - (tid / tiles_x) * tiles_x;
    const int px = tx * TILE + (threadIdx.x & 15), py = ty * TILE + (threadIdx.x >> 4);
    const bool inside = px < W && py < H;
    const int e0 = offsets[tl], e1 = offsets[tl + 1];
    const T fpx = (T)px, fpy = (T)py;
    T t = 1, cr = 0, cg = 0, cb = 0;
    int count = 0, last = 0, iters = 0;
    bool done = !inside;
    for (int base = e0; base < e1; base += FWD_BATCH) {
        if (__syncthreads_count(done) == THREADS) break;
        const int e = base + threadIdx.x;
        if (e < e1) {
            const int rank = entries[e];
            SplatF<T> s = load_splat(feat, rank);
            s_mx[threadIdx.x] = s.mx; s_my[threadIdx.x] = s.my;
            s_a[threadIdx.x] = s.a; s_b[threadIdx.x] = s.b; s_c[threadIdx.x] = s.c;
            s_op[threadIdx.x] = s.op; s_thr[threadIdx.x] = skip_threshold(s.op);
            s_r[threadIdx.x] = s.r; s_g[threadIdx.x] = s.g; s_bl[threadIdx.x] = s.bl;
            if (TOUCH) s_rank[threadIdx.x] = rank;
        }
        __syncthreads();
        const int nb = min(FWD_BATCH, e1 - base);
        if (!done) {
            for (int j = 0; j < nb; j++) {
                T d0, d1, g, alpha;
                if (!pair_eval(fpx, fpy, s_mx[j], s_my[j], s_a[j], s_b[j], s_c[j], s_op[j],
                               s_thr[j], d0, d1, g, alpha))
                    continue;
                const T test = t * ((T)1 - alpha);
                if (test < (T)T_STOP) {
                    done = true;
                    iters = base - e0 + j + 1;
                    break;
                }
                cr += s_r[j] * alpha * t;
                cg += s_g[j] * alpha * t;
                cb += s_bl[j] * alpha * t;
                t = test;
                count++;
                last = base - e0 + j + 1;
                if (TOUCH) atomicAdd((unsigned long long *)&touched[s_rank[j]], 1ull);
            }
        }
    }
    if (inside) {
        const int64_t pix = (int64_t)py * W + px;
        if (image_f64) {
            double *im = (double *)image + 3 * pix;
            im[0] = (double)(cr + t * bg0);
            im[1] = (double)(cg + t * bg1);
            im[2] = (double)(cb + t * bg2);
        } else {
            float *im = (float *)image + 3 * pix;
            im[0] = (float)(cr + t * bg0);
            im[1] = (float)(cg + t * bg1);
            im[2] = (float)(cb + t * bg2);
        }
        t_final[pix] = t;
        n_last[pix] = last;
        if (n_contrib) n_contrib[pix] = count;
        if (n_iter) n_iter[pix] = done ? iters : e1 - e0;
    }
}

// -------------------------------------------------------------- backward ----
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <typename T, typename DL>
__global__ void __launch_bounds__(THREADS) raster_bwd_kernel(
    int W, int H, int tiles_x, int row_lo, int row_hi, const int32_t *__restrict__ tile_ids,
    const int32_t *__restrict__ offsets, const int32_t *__restrict__ entries,
    const T *__restrict__ feat,
    const int4 *__restrict__ rect_sorted, const int64_t *__restrict__ emit_off, T bg0, T bg1,
    T bg2, const T *__restrict__ t_final, const int32_t *__restrict__ n_last,
    const DL *__restrict__ dl, T *__restrict__ partials) {
    __shared__ T s_mx[BWD_BATCH], s_my[BWD_BATCH], s_a[BWD_BATCH], s_b[BWD_BATCH],
        s_c[BWD_BATCH], s_op[BWD_BATCH], s_thr[BWD_BATCH], s_r[BWD_BATCH], s_g[BWD_BATCH],
        s_bl[BWD_BATCH];
    __shared__ int64_t s_slot[BWD_BATCH];
    __shared__ T s_red[WARPS][BWD_BATCH][9];
    __shared__ int s_max[WARPS];
    const int tl = blockIdx.x;
    const int tid = tile_ids ? tile_ids[tl] : row_lo * tiles_x + tl;
    const int ty = tid / tiles_x, tx = tid - (tid / tiles_x) * tiles_x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int px = tx * TILE + (threadIdx.x & 15), py = ty * TILE + (threadIdx.x >> 4);
    const bool inside = px < W && py < H;
    const int e0 = offsets[tl], e1 = offsets[tl + 1];
    const T fpx = (T)px, fpy = (T)py;
    int last = 0;
    T tn = 0, wr = 0, wg = 0, wb = 0;
    if (inside) {
        const int64_t pix = (int64_t)py * W + px;
        last = n_last[pix];
        tn = t_final[pix];
        wr = (T)dl[3 * pix];
        wg = (T)dl[3 * pix + 1];
        wb = (T)dl[3 * pix + 2];
    }
    T sr = tn * bg0, sg = tn * bg1, sb = tn * bg2;  // colour behind, bg included
    int m = last;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) s_max[warp] = m;
    __syncthreads();
    int max_last = 0;
#pragma unroll
    for (int w = 0; w < WARPS; w++) max_last = max(max_last, s_max[w]);
    const int n_ent = e1 - e0;

    // Batches cover entry indices [start, end) of the tile list, walked back
    // to front; the trailing entries [max_last, n_ent) got no contribution
    // from any pixel and receive zero subtotals.
    const int n_batches_work = (max_last + BWD_BATCH - 1) / BWD_BATCH;
    const int n_batches_all = (n_ent + BWD_BATCH - 1) / BWD_BATCH;
    for (int bi = n_batches_all - 1; bi >= 0; bi--) {
        const int start = bi * BWD_BATCH;
        const int end = min(start + BWD_BATCH, n_ent);
        __syncthreads();
        if (threadIdx.x < end - start) {
            const int rank = entries[e0 + start + threadIdx.x];
            if (emit_off) {
                const int4 rc = rect_sorted[rank];
                const int y0 = max(rc.y, row_lo);
                s_slot[threadIdx.x] =
                    emit_off[rank] + (int64_t)(ty - y0) * (rc.z - rc.x + 1) + (tx - rc.x);
            } else {
                s_slot[threadIdx.x] = (int64_t)e0 + start + threadIdx.x;
            }
            if (bi < n_batches_work) {
                SplatF<T> s = load_splat(feat, rank);
                s_mx[threadIdx.x] = s.mx; s_my[threadIdx.x] = s.my;
                s_a[threadIdx.x] = s.a; s_b[threadIdx.x] = s.b; s_c[threadIdx.x] = s.c;
                s_op[threadIdx.x] = s.op; s_thr[threadIdx.x] = skip_threshold(s.op);
                s_r[threadIdx.x] = s.r; s_g[threadIdx.x] = s.g; s_bl[threadIdx.x] = s.bl;
            }
        }
        __syncthreads();
        if (bi < n_batches_work) {
            for (int j = end - 1; j >= start; j--) {
                const int lj = j - start;
                T v[9];
#pragma unroll
                for (int k = 0; k < 9; k++) v[k] = 0;
                bool contrib = false;
                if (j < last) {
                    T d0, d1, g, alpha;
                    if (pair_eval(fpx, fpy, s_mx[lj], s_my[lj], s_a[lj], s_b[lj], s_c[lj],
                                  s_op[lj], s_thr[lj], d0, d1, g, alpha)) {
                        contrib = true;
                        const T om = (T)1 - alpha;
                        const T ti = tn / om;  // T before this splat
                        const T at = alpha * ti;
                        const T cr = s_r[lj], cg = s_g[lj], cb = s_bl[lj];
                        v[5] = wr * at;
                        v[6] = wg * at;
                        v[7] = wb * at;
                        const T dalpha = (wr * (cr * ti - sr / om) + wg * (cg * ti - sg / om) +
                                          wb * (cb * ti - sb / om));
                        sr += cr * at;
                        sg += cg * at;
                        sb += cb * at;
                        const T op = s_op[lj];
                        if (!(op * g > (T)ALPHA_CLAMP)) {
                            const T dg = dalpha * op;
                            v[8] = dalpha * g;
                            const T dpower = dg * g;
                            v[2] = dpower * ((T)-0.5 * d0 * d0);
                            v[3] = dpower * (-(d0 * d1));
                            v[4] = dpower * ((T)-0.5 * d1 * d1);
                            v[0] = dpower * (s_a[lj] * d0 + s_b[lj] * d1);
                            v[1] = dpower * (s_b[lj] * d0 + s_c[lj] * d1);
                        }
                        tn = ti;
                    }
                }
                if (__any_sync(0xffffffffu, contrib)) {
#pragma unroll
                    for (int k = 0; k < 9; k++) v[k] = warp_sum(v[k]);
                }
                if (lane == 0) {
#pragma unroll
                    for (int k = 0; k < 9; k++) s_red[warp][lj][k] = v[k];
                }
            }
        }
        __syncthreads();
        // Fixed-order fold over the 8 warps (rows 0-1, 2-3, ... of the tile).
        for (int idx = threadIdx.x; idx < (end - start) * 9; idx += THREADS) {
            const int lj = idx / 9, k = idx - lj * 9;
            T acc = 0;
            if (bi < n_batches_work) {
#pragma unroll
                for (int w = 0; w < WARPS; w++) acc += s_red[w][lj][k];
            }
            partials[9 * s_slot[lj] + k] = acc;
        }
    }
}

// ------------------------------------------------------------ fold ----------
template <typename T>
__global__ void __launch_bounds__(256) reduce_ordered_kernel(
    int64_t m, const int64_t *__restrict__ emit_off, const T *__restrict__ partials,
    const int32_t *__restrict__ order, const int4 *__restrict__ rect_sorted, int row_lo,
    int row_hi, int canon_rows, double *__restrict__ grad2d, double *__restrict__ grad_norm) {
    // One thread per rank: its slots are contiguous and already in ascending
    // tile order; they are folded sequentially (block sums when canon_rows > 0).
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    double acc[9];
    fold_rank<T>(partials, emit_off[r], emit_off[r + 1], rect_sorted, r, row_lo, canon_rows, acc);
    const int64_t row = order ? (int64_t)order[r] : r;
    double *dst = grad2d + 9 * row;
#pragma unroll
    for (int k = 0; k < 9; k++) dst[k] = acc[k];
    if (grad_norm) grad_norm[row] = hypot(acc[0], acc[1]);
}

// float32 subtotals: every warp folds 32 consecutive ranks, whose slots form
// one contiguous span (emit_off is monotone).  The span streams through two
// per-warp shared buffers with TMA bulk copies (cp.async.bulk, completion on
// an mbarrier): chunk k+1 lands while the lanes fold chunk k, each lane its
// own slots -- the same FoldState arithmetic as fold_rank.  No block barriers.
#ifndef RED_WARPS_N
#define RED_WARPS_N 4
#endif
constexpr int RED_WARPS = RED_WARPS_N;
constexpr int RED_THREADS = 32 * RED_WARPS;
#ifndef RED_SLOTS_N
#define RED_SLOTS_N 96
#endif
constexpr int RED_SLOTS = RED_SLOTS_N;  // slots per chunk (4.5 KB)

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar)),
                 "r"(count)
                 : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, unsigned bytes,
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
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
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

template <bool LIVE>
__global__ void __launch_bounds__(RED_THREADS) reduce_ordered_f32_kernel(
    int64_t m, const int64_t *__restrict__ emit_off, const float *__restrict__ partials,
    const int32_t *__restrict__ order, const int4 *__restrict__ rect_sorted, int row_lo,
    int row_hi, int canon_rows, double *__restrict__ grad2d, double *__restrict__ grad_norm) {
    constexpr int PS = partial_stride<float>();
    __shared__ __align__(128) float sbuf[RED_WARPS][2][RED_SLOTS * PS];
    __shared__ __align__(8) uint64_t sbar[RED_WARPS][2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r0 = ((int64_t)blockIdx.x * RED_WARPS + warp) * 32;
    if (r0 >= m) return;
    const int64_t r = r0 + lane;
    const bool live = r < m;
    const int64_t span0 = emit_off[r0];
    const int64_t span1 = emit_off[min(r0 + 32, m)];
    int64_t p = live ? emit_off[r] : 0;
    const int64_t p1 = live ? emit_off[r + 1] : 0;
    typename std::conditional<LIVE, FoldLive, FoldState>::type st;
    if constexpr (LIVE) {
        if (live) st.init(rect_sorted, r, row_lo, row_hi, canon_rows);
    } else {
        st.init(rect_sorted, r, live ? p1 - p : 0, row_lo, canon_rows);
    }
    const int nch = (int)((span1 - span0 + RED_SLOTS - 1) / RED_SLOTS);
    float(*buf)[RED_SLOTS * PS] = sbuf[warp];
    uint64_t *bar = sbar[warp];
    auto issue = [&](int k) {
        const int64_t c0 = span0 + (int64_t)k * RED_SLOTS;
        const unsigned n = (unsigned)min((int64_t)RED_SLOTS, span1 - c0);
        bulk_load(buf[k & 1], partials + PS * c0, n * PS * (unsigned)sizeof(float), &bar[k & 1]);
    };
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (nch > 0) issue(0);
        if (nch > 1) issue(1);
    }
    __syncwarp();
    for (int k = 0; k < nch; k++) {
        mbar_wait(&bar[k & 1], (unsigned)((k >> 1) & 1));
        const int64_t c0 = span0 + (int64_t)k * RED_SLOTS;
        const int64_t e = min(p1, c0 + RED_SLOTS);
        const float *b = buf[k & 1];
        for (; p < e; p++) st.step(b + PS * (p - c0));
        __syncwarp();
        if (lane == 0 && k + 2 < nch) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(k + 2);
        }
    }
    if (!live) return;
    st.finish();
    // order == NULL: rank-ordered output (coalesced; row-parallel consumers
    // find their rank through isg_rank_of).  Row-ordered writes of 72-byte
    // records scatter partial sectors over HBM.
    const int64_t row = order ? (int64_t)order[r] : r;
    double *dst = grad2d + 9 * row;
#pragma unroll
    for (int k = 0; k < 9; k++) dst[k] = st.acc[k];
    if (grad_norm) grad_norm[row] = hypot(st.acc[0], st.acc[1]);
}

}  // namespace isg

using namespace isg;

static int raster_fwd(int32_t feat_dtype, int32_t width, int32_t height, int32_t tiles_x,
                      int32_t row_lo, int32_t row_hi, const int32_t *tile_ids, int32_t n_tile_ids,
                      const int32_t *tile_order,
                      const int32_t *offsets, const int32_t *entries, const void *feat_sorted,
                      const double *bg, void *image, int32_t image_dtype, void *t_final,
                      int32_t *n_last, int32_t *n_contrib, int32_t *n_iter, int64_t *touched,
                      uint32_t *cmask, const isg_chunks *chunks, const int32_t *slot_rank,
                      void *stream) {
    if (width <= 0 || height <= 0 || tiles_x <= 0 || row_lo < 0 || row_hi < row_lo || !bg ||
        !image || !t_final || !n_last || n_tile_ids < 0)
        return (int)cudaErrorInvalidValue;
    const int n_tiles = tile_ids ? n_tile_ids : (row_hi - row_lo) * tiles_x;
    if (n_tiles == 0) return 0;
    cudaStream_t s = (cudaStream_t)stream;
    const int img64 = image_dtype == ISG_F64 ? 1 : 0;
    if (feat_dtype == ISG_F32) {
        launch_raster_fwd_f32(n_tiles, width, height, tiles_x, row_lo, tile_ids, tile_order,
                              offsets, entries,
                              (const float *)feat_sorted, (float)bg[0], (float)bg[1],
                              (float)bg[2], image, img64, (float *)t_final, n_last, n_contrib,
                              n_iter, touched, cmask, chunks, slot_rank, s);
    } else if (feat_dtype == ISG_F64) {
        if (touched)
            raster_fwd_kernel<double, true><<<n_tiles, THREADS, 0, s>>>(
                width, height, tiles_x, row_lo, tile_ids, offsets, entries, (const double *)feat_sorted,
                bg[0], bg[1], bg[2], image, img64, (double *)t_final, n_last, n_contrib, n_iter, touched);
        else
            raster_fwd_kernel<double, false><<<n_tiles, THREADS, 0, s>>>(
                width, height, tiles_x, row_lo, tile_ids, offsets, entries, (const double *)feat_sorted,
                bg[0], bg[1], bg[2], image, img64, (double *)t_final, n_last, n_contrib, n_iter, touched);
    } else {
        return (int)cudaErrorInvalidValue;
    }
    ISG_CHECK_LAUNCH();
    return 0;
}

static int raster_bwd(int32_t feat_dtype, int32_t width, int32_t height, int32_t tiles_x,
                      int32_t row_lo, int32_t row_hi, const int32_t *tile_ids, int32_t n_tile_ids,
                      const int32_t *tile_order,
                      const int32_t *offsets, const int32_t *entries, const void *feat_sorted,
                      const int32_t *rect_sorted, const int64_t *emit_off, const double *bg,
                      const void *t_final, const int32_t *n_last, const void *dl_dimage,
                      int32_t dl_dtype, void *partials, const uint32_t *cmask,
                      const isg_chunks *chunks, const int32_t *slot_rank, void *stream) {
    if (width <= 0 || height <= 0 || tiles_x <= 0 || row_lo < 0 || row_hi < row_lo || !bg ||
        n_tile_ids < 0 || (emit_off && !rect_sorted))
        return (int)cudaErrorInvalidValue;
    const int n_tiles = tile_ids ? n_tile_ids : (row_hi - row_lo) * tiles_x;
    if (n_tiles == 0) return 0;
    cudaStream_t s = (cudaStream_t)stream;
    const int4 *rs = (const int4 *)rect_sorted;
#define ISG_BWD(T, DL)                                                                       \
    raster_bwd_kernel<T, DL><<<n_tiles, THREADS, 0, s>>>(                                    \
        width, height, tiles_x, row_lo, row_hi, tile_ids, offsets, entries,                   \
        (const T *)feat_sorted, rs,                                                           \
        emit_off, (T)bg[0], (T)bg[1], (T)bg[2], (const T *)t_final, n_last,                  \
        (const DL *)dl_dimage, (T *)partials)
    if (feat_dtype == ISG_F32 && dl_dtype == ISG_F32)
        launch_raster_bwd_f32<float>(n_tiles, width, height, tiles_x, row_lo, tile_ids,
                                     tile_order, offsets,
                                     entries, (const float *)feat_sorted, rs, emit_off,
                                     (float)bg[0], (float)bg[1], (float)bg[2],
                                     (const float *)t_final, n_last, (const float *)dl_dimage,
                                     (float *)partials, cmask, chunks, slot_rank, s);
    else if (feat_dtype == ISG_F32 && dl_dtype == ISG_F64)
        launch_raster_bwd_f32<double>(n_tiles, width, height, tiles_x, row_lo, tile_ids,
                                      tile_order, offsets,
                                      entries, (const float *)feat_sorted, rs, emit_off,
                                      (float)bg[0], (float)bg[1], (float)bg[2],
                                      (const float *)t_final, n_last, (const double *)dl_dimage,
                                      (float *)partials, cmask, chunks, slot_rank, s);
    else if (feat_dtype == ISG_F64 && dl_dtype == ISG_F32) ISG_BWD(double, float);
    else if (feat_dtype == ISG_F64 && dl_dtype == ISG_F64) ISG_BWD(double, double);
    else return (int)cudaErrorInvalidValue;
#undef ISG_BWD
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_reduce_ordered(int32_t feat_dtype, int64_t m, const int64_t *emit_off,
                                  const void *partials, const int32_t *order,
                                  const int32_t *rect_sorted, int32_t row_lo, int32_t row_hi,
                                  int32_t canon_rows, double *grad2d, double *grad_norm,
                                  void *stream) {
    if (m < 0 || (canon_rows > 0 && !rect_sorted)) return (int)cudaErrorInvalidValue;
    const int4 *rs = (const int4 *)rect_sorted;
    if (m == 0) return 0;
    cudaStream_t s = (cudaStream_t)stream;
    if (feat_dtype == ISG_F32)
        reduce_ordered_f32_kernel<false><<<blocks_for(m, RED_THREADS), RED_THREADS, 0, s>>>(
            m, emit_off, (const float *)partials, order, rs, row_lo, row_hi, canon_rows, grad2d,
            grad_norm);
    else if (feat_dtype == ISG_F64)
        reduce_ordered_kernel<double><<<blocks_for(m, 256), 256, 0, s>>>(
            m, emit_off, (const double *)partials, order, rs, row_lo, row_hi, canon_rows, grad2d,
            grad_norm);
    else
        return (int)cudaErrorInvalidValue;
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_reduce_live(int64_t m, const int64_t *live_off, const float *partials,
                               const int32_t *order, const int32_t *rect_sorted, int32_t row_lo,
                               int32_t row_hi, int32_t canon_rows, double *grad2d,
                               double *grad_norm, void *stream) {
    if (m < 0 || canon_rows < 1 || (m > 0 && (!live_off || !partials || !rect_sorted || !grad2d)))
        return (int)cudaErrorInvalidValue;
    if (m == 0) return 0;
    reduce_ordered_f32_kernel<true><<<blocks_for(m, RED_THREADS), RED_THREADS, 0,
                                      (cudaStream_t)stream>>>(
        m, live_off, partials, order, (const int4 *)rect_sorted, row_lo, row_hi, canon_rows,
        grad2d, grad_norm);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_raster_fwd(int32_t feat_dtype, int32_t width, int32_t height, int32_t tiles_x,
                              int32_t row_lo, int32_t row_hi, const int32_t *tile_ids,
                              int32_t n_tile_ids, const int32_t *offsets,
                              const int32_t *entries, const void *feat_sorted, const double *bg,
                              void *image, int32_t image_dtype, void *t_final, int32_t *n_last,
                              int32_t *n_contrib, int32_t *n_iter, int64_t *touched,
                              void *stream) {
    return raster_fwd(feat_dtype, width, height, tiles_x, row_lo, row_hi, tile_ids, n_tile_ids,
                      nullptr,
                      offsets, entries, feat_sorted, bg, image, image_dtype, t_final, n_last,
                      n_contrib, n_iter, touched, nullptr, nullptr, nullptr, stream);
}

extern "C" int isg_raster_bwd(int32_t feat_dtype, int32_t width, int32_t height, int32_t tiles_x,
                              int32_t row_lo, int32_t row_hi, const int32_t *tile_ids,
                              int32_t n_tile_ids, const int32_t *offsets,
                              const int32_t *entries, const void *feat_sorted,
                              const int32_t *rect_sorted, const int64_t *emit_off,
                              const double *bg, const void *t_final, const int32_t *n_last,
                              const void *dl_dimage, int32_t dl_dtype, void *partials,
                              void *stream) {
    return raster_bwd(feat_dtype, width, height, tiles_x, row_lo, row_hi, tile_ids, n_tile_ids,
                      nullptr,
                      offsets, entries, feat_sorted, rect_sorted, emit_off, bg, t_final, n_last,
                      dl_dimage, dl_dtype, partials, nullptr, nullptr, nullptr, stream);
}

namespace isg {
// Work items of the chunked backward: positions of tile_order in launch
// order, each expanded into its ceil(len / chunk) chunks.  One CTA, block
// scan over the positions in rounds of 1024.
__global__ void __launch_bounds__(1024) chunk_items_kernel(int n_tiles,
                                                           const int32_t *__restrict__ offsets,
                                                           const int32_t *__restrict__ order,
                                                           const int4 *__restrict__ tile_last,
                                                           int chunk, int split,
                                                           int2 *__restrict__ items,
                                                           int32_t *__restrict__ n_items) {
    __shared__ int swarp[32];
    __shared__ int scarry;
    if (threadIdx.x == 0) scarry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int c0 = 0; c0 < n_tiles; c0 += 1024) {
        const int p = c0 + threadIdx.x;
        int tl = 0, nc = 0;
        if (p < n_tiles) {
            tl = order ? order[p] : p;
            const int4 q = tile_last[tl];
            const int len = max(max(q.x, q.y), max(q.z, q.w));
            nc = split ? max(1, (len + chunk - 1) / chunk) : 1;
        }
        int x = nc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) swarp[warp] = x;
        __syncthreads();
        int before = scarry;
        for (int w = 0; w < warp; w++) before += swarp[w];
        const int ex = before + x - nc;
        for (int k = 0; k < nc; k++) items[ex + k] = make_int2(tl, k | (k + 1 == nc ? 1 << 30 : 0));
        __syncthreads();
        if (threadIdx.x == 1023) scarry = before + x;
        __syncthreads();
    }
    if (threadIdx.x == 0) n_items[0] = scarry;
}
}  // namespace isg

extern "C" int64_t isg_chunk_state_floats(int64_t n_entries, int32_t n_tiles, int32_t chunk) {
    if (chunk <= 0 || n_entries < 0 || n_tiles < 0) return 0;
    return 4 * 256 * (n_entries / chunk + (int64_t)n_tiles + 2);
}

extern "C" int32_t isg_chunk_items_max(int64_t n_entries, int32_t n_tiles, int32_t chunk) {
    if (chunk <= 0 || n_entries < 0 || n_tiles < 0) return n_tiles;
    return (int32_t)(n_entries / chunk + (int64_t)n_tiles + 1);
}

extern "C" int isg_chunk_items(int32_t n_tiles, const int32_t *offsets, const int32_t *tile_order,
                               const int32_t *tile_last, int32_t chunk, int32_t split,
                               int32_t *items, int32_t *n_items, void *stream) {
    if (n_tiles < 0 || chunk <= 0 || chunk % 32 || !items || !n_items ||
        (n_tiles && (!offsets || !tile_last)))
        return (int)cudaErrorInvalidValue;
    chunk_items_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(
        n_tiles, offsets, tile_order, (const int4 *)tile_last, chunk, split, (int2 *)items,
        n_items);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int64_t isg_contrib_mask_words(int64_t n_entries, int32_t n_tiles) {
    if (n_entries < 0 || n_tiles < 0) return -1;
    return 4 * ((n_entries >> 5) + (int64_t)n_tiles + 1);
}

extern "C" int isg_raster_fwd_masked(int32_t width, int32_t height, int32_t tiles_x,
                                     int32_t row_lo, int32_t row_hi, const int32_t *tile_ids,
                                     int32_t n_tile_ids, const int32_t *tile_order,
                                     const int32_t *offsets,
                                     const int32_t *entries, const void *feat_sorted,
                                     const double *bg, void *image, int32_t image_dtype,
                                     void *t_final, int32_t *n_last, int32_t *n_contrib,
                                     int32_t *n_iter, int64_t *touched, uint32_t *contrib_mask,
                                     const isg_chunks *chunks, const int32_t *slot_rank,
                                     void *stream) {
    if (!contrib_mask) return (int)cudaErrorInvalidValue;
    return raster_fwd(ISG_F32, width, height, tiles_x, row_lo, row_hi, tile_ids, n_tile_ids,
                      tile_order,
                      offsets, entries, feat_sorted, bg, image, image_dtype, t_final, n_last,
                      n_contrib, n_iter, touched, contrib_mask, chunks, slot_rank, stream);
}

extern "C" int isg_raster_bwd_masked(int32_t width, int32_t height, int32_t tiles_x,
                                     int32_t row_lo, int32_t row_hi, const int32_t *tile_ids,
                                     int32_t n_tile_ids, const int32_t *tile_order,
                                     const int32_t *offsets,
                                     const int32_t *entries, const void *feat_sorted,
                                     const int32_t *rect_sorted, const int64_t *emit_off,
                                     const double *bg, const void *t_final,
                                     const int32_t *n_last, const void *dl_dimage,
                                     int32_t dl_dtype, void *partials,
                                     const uint32_t *contrib_mask, const isg_chunks *chunks,
                                     const int32_t *slot_rank, void *stream) {
    if (!contrib_mask || (dl_dtype != ISG_F32 && dl_dtype != ISG_F64))
        return (int)cudaErrorInvalidValue;
    return raster_bwd(ISG_F32, width, height, tiles_x, row_lo, row_hi, tile_ids, n_tile_ids,
                      tile_order,
                      offsets, entries, feat_sorted, rect_sorted, emit_off, bg, t_final, n_last,
                      dl_dimage, dl_dtype, partials, contrib_mask, chunks, slot_rank, stream);
}
