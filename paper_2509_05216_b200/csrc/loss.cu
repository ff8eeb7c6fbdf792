// loss.cu -- fused L1 + D-SSIM loss and its exact image gradient (sm_100a).
//
// metrics.py:135-189.  Two separable stencil passes, each staged through
// shared memory in 16x64 output tiles with a 10-pixel halo:
//   1. fields  -- per valid centre and channel: the five 11x11 Gaussian
//                 moments (rows then columns, like _corr_valid), SSIM p*q and
//                 the three adjoint fields f0, f1, f2 (metrics.py:166-183);
//   2. adjoint -- per pixel: the adjoint correlation of f0..f2 (zero outside
//                 the valid region, like _corr_adjoint), combined with the L1
//                 sign term into dL/dimage.
// Both passes work on a band of image rows [row0, row1) (multiples of 16), so
// a GPU that renders one row band computes its pixels' gradient from its band
// plus a halo (16 rows above, 10 below).  Loss partials are written per 16x16
// block into arrays indexed over the FULL image; every block is owned by
// exactly one band, and the final sum runs over the full arrays in a fixed
// order -- so the loss is identical for any band split.
#include "common.cuh"

namespace isg {

// metrics._W1D, pinned bit for bit (tests/test_oracle_golden.py).
__constant__ double c_w1d[11] = {
    0x1.0d956b52a1d70p-10, 0x1.f1fe01ae5a5b8p-8, 0x1.26eb175d83f67p-5,
    0x1.bff0fe8e98418p-4,  0x1.b43c3f52b19f2p-3, 0x1.106560aa892c0p-2,
    0x1.b43c3f52b19f2p-3,  0x1.bff0fe8e98418p-4, 0x1.26eb175d83f67p-5,
    0x1.f1fe01ae5a5b8p-8,  0x1.0d956b52a1d70p-10};
__constant__ float c_w1f[11] = {
    (float)0x1.0d956b52a1d70p-10, (float)0x1.f1fe01ae5a5b8p-8, (float)0x1.26eb175d83f67p-5,
    (float)0x1.bff0fe8e98418p-4,  (float)0x1.b43c3f52b19f2p-3, (float)0x1.106560aa892c0p-2,
    (float)0x1.b43c3f52b19f2p-3,  (float)0x1.bff0fe8e98418p-4, (float)0x1.26eb175d83f67p-5,
    (float)0x1.f1fe01ae5a5b8p-8,  (float)0x1.0d956b52a1d70p-10};

template <typename T> __device__ __forceinline__ T wt(int i);
template <> __device__ __forceinline__ float wt<float>(int i) { return c_w1f[i]; }
template <> __device__ __forceinline__ double wt<double>(int i) { return c_w1d[i]; }

// float32 instantiation: two consecutive outputs of a stencil row accumulate
// as one packed pair (fma.rn.f32x2 -> FFMA2, each component the scalar FMA):
// output pair (o, o + 1) takes input i with the weight pair (w[i - o],
// w[i - o - 1]), zero past either end of the 11 taps.  Every accumulator is a
// sum of products whose exact value is never a negative zero, so the extra
// zero-weight FMA at a pair's edge (acc + 0 * v) leaves it bit for bit, and
// each output still sums its taps in ascending order.
#ifndef LOSS_PACK2
#define LOSS_PACK2 1
#endif
typedef unsigned long long lf2_t;
__device__ __forceinline__ lf2_t lpk(float a, float b) {
    lf2_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void lup(lf2_t r, float &a, float &b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ lf2_t lfma2(lf2_t a, lf2_t b, lf2_t c) {
    lf2_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
// weight pair for tap t of the pair's first output (t in [0, 11]):
// (w[t], w[t - 1]), 64-bit constants the FFMA2 reads from the constant bank
#define W1F(i) ((float)c_w1d_host[i])
constexpr double c_w1d_host[11] = {
    0x1.0d956b52a1d70p-10, 0x1.f1fe01ae5a5b8p-8, 0x1.26eb175d83f67p-5,
    0x1.bff0fe8e98418p-4,  0x1.b43c3f52b19f2p-3, 0x1.106560aa892c0p-2,
    0x1.b43c3f52b19f2p-3,  0x1.bff0fe8e98418p-4, 0x1.26eb175d83f67p-5,
    0x1.f1fe01ae5a5b8p-8,  0x1.0d956b52a1d70p-10};
__constant__ float2 c_w2f[12] = {
    {W1F(0), 0.0f},    {W1F(1), W1F(0)}, {W1F(2), W1F(1)}, {W1F(3), W1F(2)},
    {W1F(4), W1F(3)},  {W1F(5), W1F(4)}, {W1F(6), W1F(5)}, {W1F(7), W1F(6)},
    {W1F(8), W1F(7)},  {W1F(9), W1F(8)}, {W1F(10), W1F(9)}, {0.0f, W1F(10)}};
#undef W1F
__device__ __forceinline__ lf2_t wpair(int t) {
    return *reinterpret_cast<const lf2_t *>(&c_w2f[t]);
}

// Ground-truth sample: float/double as stored, or an 8-bit code k read as
// float(k / 255.0) -- the value the reference's PNG load + astype produces.
template <typename T, typename R>
__device__ __forceinline__ T gt_val(R v) { return (T)v; }
template <>
__device__ __forceinline__ float gt_val<float, uint8_t>(uint8_t v) { return (float)((double)v / 255.0); }
template <>
__device__ __forceinline__ double gt_val<double, uint8_t>(uint8_t v) { return (double)v / 255.0; }

constexpr int LT = 16;          // output tile edge
constexpr int LP = LT + 10;     // patch edge (tile + 10-px halo)

// 8-bit ground truth: the 256 values float(k / 255.0) (gt_val) staged once per
// block in shared memory, so a sample costs one shared load instead of a
// float64 division.
template <typename T, typename R>
struct GtLut {
    __device__ __forceinline__ void init(T *) const {}
    __device__ __forceinline__ T operator()(const T *, R v) const { return gt_val<T, R>(v); }
};
template <typename T>
struct GtLut<T, uint8_t> {
    __device__ __forceinline__ void init(T *lut) const {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) lut[i] = gt_val<T, uint8_t>((uint8_t)i);
    }
    __device__ __forceinline__ T operator()(const T *lut, uint8_t v) const { return lut[v]; }
};

__device__ __forceinline__ double block_sum(double v, double *scratch) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += scratch[w];
    return s;
}

// Both passes run on 16-row x 64-column output tiles (LT x FW) with the
// 10-pixel halo staged in shared memory (dynamic, FPH x FPW per plane).  The
// separable 11-tap correlations are register-tiled: the horizontal pass gives
// each of 208 threads one patch row and HK = 8 consecutive outputs (18 loads
// feed 88 taps), the vertical pass gives each of 256 threads one column and
// VK = 4 consecutive rows.  Every output still sums its taps in ascending
// order, exactly as _corr_valid / _corr_adjoint do.  Partials stay per 16x16
// block (4 per tile, each reduced in a fixed order), so the loss is
// independent of the row-band split.
constexpr int FW = 64;          // output tile width
constexpr int FPW = FW + 10;    // patch width
constexpr int FPH = LT + 10;    // patch height
constexpr int HK = 8;           // horizontal outputs per thread
constexpr int VK = 4;           // vertical outputs per thread
constexpr int HTASKS = FPH * (FW / HK);  // 208
constexpr int PR = (FPH + 7) / 8;          // patch rows per warp (8 warps)
constexpr int PC = (FPW + 31) / 32;        // patch columns per lane
constexpr int LTHREADS = 256;
static_assert(LTHREADS == FW * (LT / VK), "vertical pass covers the tile");

// Sum of a double over the 16 lanes of each half warp, then over the 4
// row-runs of a 16x16 sub-block in fixed order; returns the sub-block sum
// for threads 0..3 (sub-block = threadIdx.x).
__device__ __forceinline__ double subblock_sum(double v, double *red /* [4][4] */) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int col = threadIdx.x & (FW - 1), rr = threadIdx.x / FW;
    if ((threadIdx.x & 15) == 0) red[rr * 4 + (col >> 4)] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x < 4)
        for (int r = 0; r < LT / VK; r++) s += red[r * 4 + threadIdx.x];
    return s;
}

// Pass 1 over centre block rows by_base + blockIdx.y.  img/ref are indexed by
// global row (img points at global row img_row0).  fmap (may be NULL) holds
// centre rows from fmap_row0: layout [field][channel][rows][wc].  Partials are
// written for centre blocks whose first row lies in [own0, own1), indexed by
// 16x16 centre block over the full image.
template <typename T, typename IN, typename R>
#ifndef LF_MINB
#define LF_MINB 4
#endif
__global__ void __launch_bounds__(LTHREADS, LF_MINB) ssim_fields_kernel(
    int H, int W, int C, const IN *__restrict__ img, int img_row0, const R *__restrict__ ref,
    T *__restrict__ fmap, int fmap_row0, int fmap_rows, int by_base, int own0, int own1,
    double *__restrict__ part) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T(*sx)[FPW] = reinterpret_cast<T(*)[FPW]>(smem_raw);
    T(*sy)[FPW] = sx + FPH;
    T(*hs)[FPH][FW] = reinterpret_cast<T(*)[FPH][FW]>(sy + FPH);  // [5]
    __shared__ double red[16];
    __shared__ T lut[256];
    const GtLut<T, R> gt;
    gt.init(lut);
    const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;  // == pow(0.01, 2), pow(0.03, 2)
    const int hc = H - 10, wc = W - 10;
    const int by = by_base + blockIdx.y;
    const int cx0 = blockIdx.x * FW, cy0 = by * LT;
    const int col = threadIdx.x & (FW - 1), rr = threadIdx.x / FW;
    const int ccx = cx0 + col;
    const int hr = threadIdx.x >> 3, hu = threadIdx.x & 7;  // horizontal task
    const int lwarp = threadIdx.x >> 5, llane = threadIdx.x & 31;
    double pq_acc = 0.0;
    __syncthreads();
    for (int c = 0; c < C; c++) {
        {
            // warp w stages patch rows w, w+8, ..; a row's loads are issued
            // before its stores
#pragma unroll 2
            for (int i = 0; i < PR; i++) {
                IN vx[PC];
                R vy[PC];
                const int r = lwarp + 8 * i, y = cy0 + r;
#pragma unroll
                for (int k = 0; k < PC; k++) {
                    const int q = llane + 32 * k, x = cx0 + q;
                    const bool ok = r < FPH && q < FPW && y < H && x < W;
                    vx[k] = ok ? img[((int64_t)(y - img_row0) * W + x) * C + c] : (IN)0;
                    vy[k] = ok ? ref[((int64_t)y * W + x) * C + c] : (R)0;
                }
#pragma unroll
                for (int k = 0; k < PC; k++) {
                    const int q = llane + 32 * k;
                    if (r < FPH && q < FPW) {
                        sx[r][q] = (T)vx[k];
                        sy[r][q] = gt(lut, vy[k]);
                    }
                }
            }
        }
        __syncthreads();
#if LOSS_PACK2
        if (sizeof(T) == 4 && threadIdx.x < HTASKS) {
            lf2_t a[5][HK / 2];
#pragma unroll
            for (int o = 0; o < HK / 2; o++)
#pragma unroll
                for (int f = 0; f < 5; f++) a[f][o] = lpk(0.0f, 0.0f);
#pragma unroll
            for (int i = 0; i < HK + 10; i++) {
                const float x = (float)sx[hr][hu * HK + i], y = (float)sy[hr][hu * HK + i];
                const float xx = x * x, yy = y * y, xy = x * y;
#pragma unroll
                for (int o = 0; o < HK / 2; o++) {
                    const int t = i - 2 * o;
                    if (t >= 0 && t <= 11) {
                        const lf2_t w = wpair(t);
                        a[0][o] = lfma2(w, lpk(x, x), a[0][o]);
                        a[1][o] = lfma2(w, lpk(y, y), a[1][o]);
                        a[2][o] = lfma2(w, lpk(xx, xx), a[2][o]);
                        a[3][o] = lfma2(w, lpk(yy, yy), a[3][o]);
                        a[4][o] = lfma2(w, lpk(xy, xy), a[4][o]);
                    }
                }
            }
#pragma unroll
            for (int f = 0; f < 5; f++)
#pragma unroll
                for (int o = 0; o < HK / 2; o++) {
                    float u, v;
                    lup(a[f][o], u, v);
                    hs[f][hr][hu * HK + 2 * o] = (T)u;
                    hs[f][hr][hu * HK + 2 * o + 1] = (T)v;
                }
        } else
#endif
        if (threadIdx.x < HTASKS) {
            T a[5][HK];
#pragma unroll
            for (int o = 0; o < HK; o++)
#pragma unroll
                for (int f = 0; f < 5; f++) a[f][o] = 0;
#pragma unroll
            for (int i = 0; i < HK + 10; i++) {
                const T x = sx[hr][hu * HK + i], y = sy[hr][hu * HK + i];
                const T xx = x * x, yy = y * y, xy = x * y;
#pragma unroll
                for (int o = 0; o < HK; o++) {
                    const int t = i - o;
                    if (t >= 0 && t < 11) {
                        const T w = wt<T>(t);
                        a[0][o] += w * x;
                        a[1][o] += w * y;
                        a[2][o] += w * xx;
                        a[3][o] += w * yy;
                        a[4][o] += w * xy;
                    }
                }
            }
#pragma unroll
            for (int f = 0; f < 5; f++)
#pragma unroll
                for (int o = 0; o < HK; o++) hs[f][hr][hu * HK + o] = a[f][o];
        }
        __syncthreads();
        {
            T m[5][VK];
#if LOSS_PACK2
            if (sizeof(T) == 4) {
                lf2_t m2[5][VK / 2];
#pragma unroll
                for (int k = 0; k < VK / 2; k++)
#pragma unroll
                    for (int f = 0; f < 5; f++) m2[f][k] = lpk(0.0f, 0.0f);
#pragma unroll
                for (int t = 0; t < VK + 10; t++) {
                    float h[5];
#pragma unroll
                    for (int f = 0; f < 5; f++) h[f] = (float)hs[f][rr * VK + t][col];
#pragma unroll
                    for (int k = 0; k < VK / 2; k++) {
                        const int i = t - 2 * k;
                        if (i >= 0 && i <= 11) {
                            const lf2_t w = wpair(i);
#pragma unroll
                            for (int f = 0; f < 5; f++) m2[f][k] = lfma2(w, lpk(h[f], h[f]), m2[f][k]);
                        }
                    }
                }
#pragma unroll
                for (int f = 0; f < 5; f++)
#pragma unroll
                    for (int k = 0; k < VK / 2; k++) {
                        float u, v;
                        lup(m2[f][k], u, v);
                        m[f][2 * k] = (T)u;
                        m[f][2 * k + 1] = (T)v;
                    }
            } else
#endif
            {
#pragma unroll
            for (int k = 0; k < VK; k++)
#pragma unroll
                for (int f = 0; f < 5; f++) m[f][k] = 0;
#pragma unroll
            for (int t = 0; t < VK + 10; t++) {
                T h[5];
#pragma unroll
                for (int f = 0; f < 5; f++) h[f] = hs[f][rr * VK + t][col];
#pragma unroll
                for (int k = 0; k < VK; k++) {
                    const int i = t - k;
                    if (i >= 0 && i < 11) {
                        const T w = wt<T>(i);
#pragma unroll
                        for (int f = 0; f < 5; f++) m[f][k] += w * h[f];
                    }
                }
            }
            }
#pragma unroll
            for (int k = 0; k < VK; k++) {
                const int ccy = cy0 + rr * VK + k;
                if (ccx < wc && ccy < hc) {
                    const T mx = m[0][k], my = m[1][k], mxx = m[2][k], myy = m[3][k],
                            mxy = m[4][k];
                    const T var_x = mxx - mx * mx, var_y = myy - my * my, cov = mxy - mx * my;
                    const T a1 = (T)2 * mx * my + (T)C1;
                    const T b1 = mx * mx + my * my + (T)C1;
                    const T a2 = (T)2 * cov + (T)C2;
                    const T b2 = var_x + var_y + (T)C2;
                    const T rb1 = (T)1 / b1, rb2 = (T)1 / b2;
                    const T p = a1 * rb1, q = a2 * rb2;
                    pq_acc += (double)(p * q);
                    if (fmap) {
                        const T dp_dmux = ((T)2 * my * b1 - (T)2 * mx * a1) * (rb1 * rb1);
                        const T d_mu = q * dp_dmux;
                        const T d_sigma = -((p * q) * rb2);
                        const T d_xy = ((T)2 * p) * rb2;
                        const T f1 = (T)2 * d_sigma, f2 = d_xy;
                        const T f0 = d_mu - f1 * mx - f2 * my;
                        const int64_t plane = (int64_t)fmap_rows * wc;
                        const int64_t o = (int64_t)(ccy - fmap_row0) * wc + ccx;
                        fmap[(0 * C + c) * plane + o] = f0;
                        fmap[(1 * C + c) * plane + o] = f1;
                        fmap[(2 * C + c) * plane + o] = f2;
                    }
                }
            }
        }
        __syncthreads();
    }
    const double s = subblock_sum(pq_acc, red);
    const int nbx = (wc + LT - 1) / LT, bx = blockIdx.x * (FW / LT) + (int)threadIdx.x;
    if (threadIdx.x < FW / LT && bx < nbx && cy0 >= own0 && cy0 < own1) part[by * nbx + bx] = s;
}

// Pass 2 over pixel block rows by_base + blockIdx.y:
// dL/dimage = sign(x-y)(1-lam)/n + gscale * (A f0 + x A f1 + y A f2).
// grad is indexed by global row from grad_row0.
template <typename T, typename IN, typename R>
#ifndef LA_MINB
#define LA_MINB 4
#endif
__global__ void __launch_bounds__(LTHREADS, LA_MINB) ssim_adjoint_kernel(
    int H, int W, const IN *__restrict__ img, int img_row0, const R *__restrict__ ref,
    const T *__restrict__ fmap, int fmap_row0, int fmap_rows, IN *__restrict__ grad,
    int grad_row0, int row1, int by_base, T l1_scale, T gscale, double *__restrict__ part) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T(*sf)[FPH][FPW] = reinterpret_cast<T(*)[FPH][FPW]>(smem_raw);            // [3]
    T(*hs)[FPH][FW] = reinterpret_cast<T(*)[FPH][FW]>(sf + 3);                // [3]
    __shared__ double red[16];
    __shared__ T lut[256];
    const GtLut<T, R> gt;
    gt.init(lut);
    const int hc = H - 10, wc = W - 10;
    const int by = by_base + blockIdx.y;
    const int x0 = blockIdx.x * FW, y0 = by * LT;
    const int col = threadIdx.x & (FW - 1), rr = threadIdx.x / FW;
    const int x = x0 + col;
    const int hr = threadIdx.x >> 3, hu = threadIdx.x & 7;
    const int lwarp = threadIdx.x >> 5, llane = threadIdx.x & 31;
    const int64_t plane = (int64_t)fmap_rows * wc;
    double l1_acc = 0.0;
    __syncthreads();
    for (int c = 0; c < 3; c++) {
        // this thread's pixels' image / ground-truth samples, loaded early
        IN xin[VK];
        R yin[VK];
#pragma unroll
        for (int k = 0; k < VK; k++) {
            const int y = y0 + rr * VK + k;
            const bool ok = x < W && y < H && y < row1;
            xin[k] = ok ? img[((int64_t)(y - img_row0) * W + x) * 3 + c] : (IN)0;
            yin[k] = ok ? ref[((int64_t)y * W + x) * 3 + c] : (R)0;
        }
#pragma unroll 2
        for (int i = 0; i < PR; i++) {
            T v[3][PC];
            const int r = lwarp + 8 * i, cy = y0 - 10 + r;
#pragma unroll
            for (int k = 0; k < PC; k++) {
                const int q = llane + 32 * k, cx = x0 - 10 + q;
                const bool ok = r < FPH && q < FPW && cy >= 0 && cy < hc && cx >= 0 && cx < wc;
                const int64_t o = (int64_t)(cy - fmap_row0) * wc + cx;
#pragma unroll
                for (int f = 0; f < 3; f++) v[f][k] = ok ? fmap[(f * 3 + c) * plane + o] : (T)0;
            }
#pragma unroll
            for (int k = 0; k < PC; k++) {
                const int q = llane + 32 * k;
                if (r < FPH && q < FPW) {
#pragma unroll
                    for (int f = 0; f < 3; f++) sf[f][r][q] = v[f][k];
                }
            }
        }
        __syncthreads();
#if LOSS_PACK2
        if (sizeof(T) == 4 && threadIdx.x < HTASKS) {
#pragma unroll
            for (int f = 0; f < 3; f++) {
                lf2_t a[HK / 2];
#pragma unroll
                for (int o = 0; o < HK / 2; o++) a[o] = lpk(0.0f, 0.0f);
#pragma unroll
                for (int i = 0; i < HK + 10; i++) {
                    const float v = (float)sf[f][hr][hu * HK + i];
#pragma unroll
                    for (int o = 0; o < HK / 2; o++) {
                        const int t = i - 2 * o;
                        if (t >= 0 && t <= 11) a[o] = lfma2(wpair(t), lpk(v, v), a[o]);
                    }
                }
#pragma unroll
                for (int o = 0; o < HK / 2; o++) {
                    float u, w;
                    lup(a[o], u, w);
                    hs[f][hr][hu * HK + 2 * o] = (T)u;
                    hs[f][hr][hu * HK + 2 * o + 1] = (T)w;
                }
            }
        } else
#endif
        if (threadIdx.x < HTASKS) {
#pragma unroll
            for (int f = 0; f < 3; f++) {
                T a[HK];
#pragma unroll
                for (int o = 0; o < HK; o++) a[o] = 0;
#pragma unroll
                for (int i = 0; i < HK + 10; i++) {
                    const T v = sf[f][hr][hu * HK + i];
#pragma unroll
                    for (int o = 0; o < HK; o++) {
                        const int t = i - o;
                        if (t >= 0 && t < 11) a[o] += wt<T>(t) * v;
                    }
                }
#pragma unroll
                for (int o = 0; o < HK; o++) hs[f][hr][hu * HK + o] = a[o];
            }
        }
        __syncthreads();
        {
            T g[3][VK];
#if LOSS_PACK2
            if (sizeof(T) == 4) {
                lf2_t g2[3][VK / 2];
#pragma unroll
                for (int k = 0; k < VK / 2; k++) g2[0][k] = g2[1][k] = g2[2][k] = lpk(0.0f, 0.0f);
#pragma unroll
                for (int t = 0; t < VK + 10; t++) {
                    const float h0 = (float)hs[0][rr * VK + t][col], h1 = (float)hs[1][rr * VK + t][col],
                                h2 = (float)hs[2][rr * VK + t][col];
#pragma unroll
                    for (int k = 0; k < VK / 2; k++) {
                        const int i = t - 2 * k;
                        if (i >= 0 && i <= 11) {
                            const lf2_t w = wpair(i);
                            g2[0][k] = lfma2(w, lpk(h0, h0), g2[0][k]);
                            g2[1][k] = lfma2(w, lpk(h1, h1), g2[1][k]);
                            g2[2][k] = lfma2(w, lpk(h2, h2), g2[2][k]);
                        }
                    }
                }
#pragma unroll
                for (int f = 0; f < 3; f++)
#pragma unroll
                    for (int k = 0; k < VK / 2; k++) {
                        float u, v;
                        lup(g2[f][k], u, v);
                        g[f][2 * k] = (T)u;
                        g[f][2 * k + 1] = (T)v;
                    }
            } else
#endif
            {
#pragma unroll
            for (int k = 0; k < VK; k++) g[0][k] = g[1][k] = g[2][k] = 0;
#pragma unroll
            for (int t = 0; t < VK + 10; t++) {
                const T h0 = hs[0][rr * VK + t][col], h1 = hs[1][rr * VK + t][col],
                        h2 = hs[2][rr * VK + t][col];
#pragma unroll
                for (int k = 0; k < VK; k++) {
                    const int i = t - k;
                    if (i >= 0 && i < 11) {
                        const T w = wt<T>(i);
                        g[0][k] += w * h0;
                        g[1][k] += w * h1;
                        g[2][k] += w * h2;
                    }
                }
            }
            }
#pragma unroll
            for (int k = 0; k < VK; k++) {
                const int y = y0 + rr * VK + k;
                if (x < W && y < H && y < row1) {
                    const T xv = (T)xin[k];
                    const T yv = gt(lut, yin[k]);
                    const T d = xv - yv;
                    const T sg = d > (T)0 ? (T)1 : (d < (T)0 ? (T)-1 : (T)0);
                    const T gg = g[0][k] + xv * g[1][k] + yv * g[2][k];
                    grad[((int64_t)(y - grad_row0) * W + x) * 3 + c] = (IN)(sg * l1_scale + gscale * gg);
                    l1_acc += (double)fabs(d);
                }
            }
        }
        __syncthreads();
    }
    const double s = subblock_sum(l1_acc, red);
    const int nbx = (W + LT - 1) / LT, bx = blockIdx.x * (FW / LT) + (int)threadIdx.x;
    if (threadIdx.x < FW / LT && bx < nbx) part[by * nbx + bx] = s;
}

template <typename T>
constexpr size_t fields_smem() { return sizeof(T) * (2 * FPH * FPW + 5 * FPH * FW); }
template <typename T>
constexpr size_t adjoint_smem() { return sizeof(T) * (3 * FPH * FPW + 3 * FPH * FW); }

// Opt the kernels into their dynamic shared memory once per process.
template <typename T, typename IN, typename R>
inline void loss_smem_optin() {
    static bool done = false;
    if (done) return;
    cudaFuncSetAttribute(ssim_fields_kernel<T, IN, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)fields_smem<T>());
    cudaFuncSetAttribute(ssim_adjoint_kernel<T, IN, R>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)adjoint_smem<T>());
    done = true;
}

// Fixed-order final reduction (one block): loss = (1-lam) L1 + lam (1 - SSIM).
// Each thread sums a strided subset in index order; the loads of a batch of
// 8 are issued together so the loop is not one dependent load per element.
constexpr int FINISH_THREADS = 1024;

__device__ __forceinline__ double strided_sum(const double *__restrict__ x, int n) {
    double a = 0.0;
    for (int i0 = threadIdx.x; i0 < n; i0 += 8 * FINISH_THREADS) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const int i = i0 + u * FINISH_THREADS;
            v[u] = i < n ? x[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; u++)
            if (i0 + u * FINISH_THREADS < n) a += v[u];
    }
    return a;
}

__global__ void __launch_bounds__(FINISH_THREADS) loss_finish_kernel(
    int n_ssim, const double *__restrict__ ssim_part, int n_l1, const double *__restrict__ l1_part,
    double n_pix, double n_centers, double lam, double *__restrict__ out) {
    __shared__ double red[FINISH_THREADS / 32];
    const double a = strided_sum(ssim_part, n_ssim);
    const double b = strided_sum(l1_part, n_l1);
    const double sa = block_sum(a, red);
    __syncthreads();
    const double sb = block_sum(b, red);
    if (threadIdx.x == 0) {
        if (n_l1 > 0)
            out[0] = (1.0 - lam) * (sb / n_pix) + lam * (1.0 - sa / n_centers);
        else
            out[0] = sa / n_centers;  // SSIM only
    }
}

inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

struct LossGrid {
    dim3 gf, ga;
    int fby0, fby1;  // centre block rows computed (incl. the halo block above)
    int aby0, aby1;  // pixel block rows
    int fmap_row0, fmap_rows;
};

inline LossGrid loss_grid(int H, int W, int row0, int row1) {
    LossGrid g;
    const int hc = H - 10, wc = W - 10;
    const int nfy = (hc + LT - 1) / LT;
    g.gf = dim3((wc + LT - 1) / LT, nfy);          // 16x16 partial blocks
    g.ga = dim3((W + LT - 1) / LT, (H + LT - 1) / LT);
    g.fby0 = row0 / LT > 0 ? row0 / LT - 1 : 0;
    g.fby1 = (row1 + LT - 1) / LT < nfy ? (row1 + LT - 1) / LT : nfy;
    if (g.fby1 < g.fby0) g.fby1 = g.fby0;
    g.aby0 = row0 / LT;
    g.aby1 = (row1 + LT - 1) / LT;
    g.fmap_row0 = g.fby0 * LT;
    g.fmap_rows = (g.fby1 - g.fby0) * LT;
    return g;
}

template <typename T, typename R>
int loss_rows_impl(void *ws, size_t *ws_bytes, int H, int W, int row0, int row1, const T *img,
                   int img_row0, const R *ref, double lam, T *grad, double *part_ssim,
                   double *part_l1, cudaStream_t s) {
    const LossGrid g = loss_grid(H, W, row0, row1);
    const int wc = W - 10;
    const size_t need = al(sizeof(T) * 9 * (size_t)(g.fmap_rows > 0 ? g.fmap_rows : 1) * wc);
    if (!ws) {
        *ws_bytes = need;
        return 0;
    }
    if (*ws_bytes < need) return (int)cudaErrorInvalidValue;
    T *fmap = (T *)ws;
    const double n_pix = 3.0 * H * W, n_centers = 3.0 * (H - 10) * (W - 10);
    loss_smem_optin<T, T, R>();
    if (g.fby1 > g.fby0) {
        dim3 grid((wc + FW - 1) / FW, g.fby1 - g.fby0);
        ssim_fields_kernel<T, T, R><<<grid, LTHREADS, fields_smem<T>(), s>>>(
            H, W, 3, img, img_row0, ref, fmap, g.fmap_row0, g.fmap_rows, g.fby0, row0, row1,
            part_ssim);
        ISG_CHECK_LAUNCH();
    }
    if (g.aby1 > g.aby0) {
        dim3 grid((W + FW - 1) / FW, g.aby1 - g.aby0);
        ssim_adjoint_kernel<T, T, R><<<grid, LTHREADS, adjoint_smem<T>(), s>>>(
            H, W, img, img_row0, ref, fmap, g.fmap_row0, g.fmap_rows, grad, row0, row1, g.aby0,
            (T)((1.0 - lam) / n_pix), (T)(-lam / n_centers), part_l1);
        ISG_CHECK_LAUNCH();
    }
    return 0;
}

template <typename T>
int loss_rows_dispatch(void *ws, size_t *ws_bytes, int H, int W, int row0, int row1,
                       const void *img, int img_row0, const void *ref, int ref_u8, double lam,
                       void *grad, double *ps, double *pl, cudaStream_t s) {
    if (ref_u8)
        return loss_rows_impl<T, uint8_t>(ws, ws_bytes, H, W, row0, row1, (const T *)img,
                                          img_row0, (const uint8_t *)ref, lam, (T *)grad, ps, pl,
                                          s);
    return loss_rows_impl<T, T>(ws, ws_bytes, H, W, row0, row1, (const T *)img, img_row0,
                                (const T *)ref, lam, (T *)grad, ps, pl, s);
}

}  // namespace isg

using namespace isg;

extern "C" int isg_loss_partials_size(int32_t height, int32_t width, int32_t *n_ssim,
                                      int32_t *n_l1) {
    if (height < 11 || width < 11 || !n_ssim || !n_l1) return (int)cudaErrorInvalidValue;
    const LossGrid g = loss_grid(height, width, 0, height);
    *n_ssim = (int32_t)(g.gf.x * g.gf.y);
    *n_l1 = (int32_t)(g.ga.x * g.ga.y);
    return 0;
}

extern "C" int isg_loss_rows(void *workspace, size_t *ws_bytes, int32_t dtype, int32_t height,
                             int32_t width, int32_t row0, int32_t row1, const void *image,
                             int32_t img_row0, const void *ref, int32_t ref_u8,
                             double lambda_dssim, void *grad, double *part_ssim, double *part_l1,
                             void *stream) {
    if (!ws_bytes || height < 11 || width < 11 || lambda_dssim < 0.0 || lambda_dssim > 1.0 ||
        row0 < 0 || row1 > height || row0 > row1 || row0 % LT != 0 ||
        (row1 % LT != 0 && row1 != height))
        return (int)cudaErrorInvalidValue;
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == ISG_F32)
        return loss_rows_dispatch<float>(workspace, ws_bytes, height, width, row0, row1, image,
                                         img_row0, ref, ref_u8, lambda_dssim, grad, part_ssim,
                                         part_l1, s);
    if (dtype == ISG_F64)
        return loss_rows_dispatch<double>(workspace, ws_bytes, height, width, row0, row1, image,
                                          img_row0, ref, ref_u8, lambda_dssim, grad, part_ssim,
                                          part_l1, s);
    return (int)cudaErrorInvalidValue;
}

extern "C" int isg_loss_finish(int32_t height, int32_t width, double lambda_dssim,
                               const double *part_ssim, const double *part_l1, double *loss_dev,
                               void *stream) {
    int32_t nf = 0, na = 0;
    int e = isg_loss_partials_size(height, width, &nf, &na);
    if (e) return e;
    const double n_pix = 3.0 * height * width, n_centers = 3.0 * (height - 10) * (width - 10);
    loss_finish_kernel<<<1, FINISH_THREADS, 0, (cudaStream_t)stream>>>(nf, part_ssim, na, part_l1, n_pix,
                                                            n_centers, lambda_dssim, loss_dev);
    ISG_CHECK_LAUNCH();
    return 0;
}

// Whole image: loss_rows(0, H) + finish, partial arrays in the workspace.
extern "C" int isg_loss_l1_dssim(void *workspace, size_t *ws_bytes, int32_t dtype, int32_t height,
                                 int32_t width, const void *image, const void *ref,
                                 int32_t ref_u8, double lambda_dssim, void *grad,
                                 double *loss_dev, void *stream) {
    if (!ws_bytes || height < 11 || width < 11 || lambda_dssim < 0.0 || lambda_dssim > 1.0)
        return (int)cudaErrorInvalidValue;
    int32_t nf = 0, na = 0;
    isg_loss_partials_size(height, width, &nf, &na);
    size_t rows_bytes = 0;
    int e = isg_loss_rows(nullptr, &rows_bytes, dtype, height, width, 0, height, nullptr, 0,
                          nullptr, ref_u8, lambda_dssim, nullptr, nullptr, nullptr, nullptr);
    if (e) return e;
    const size_t need = al(rows_bytes) + al(8 * (size_t)nf) + al(8 * (size_t)na);
    if (!workspace) {
        *ws_bytes = need;
        return 0;
    }
    if (*ws_bytes < need) return (int)cudaErrorInvalidValue;
    double *ps = (double *)((char *)workspace + al(rows_bytes));
    double *pl = (double *)((char *)ps + al(8 * (size_t)nf));
    e = isg_loss_rows(workspace, &rows_bytes, dtype, height, width, 0, height, image, 0, ref,
                      ref_u8, lambda_dssim, grad, ps, pl, stream);
    if (e) return e;
    return isg_loss_finish(height, width, lambda_dssim, ps, pl, loss_dev, stream);
}

extern "C" int isg_ssim(void *workspace, size_t *ws_bytes, int32_t height, int32_t width,
                        int32_t channels, const double *image, const double *ref,
                        double *out_dev, void *stream) {
    if (!ws_bytes || height < 11 || width < 11 || channels < 1)
        return (int)cudaErrorInvalidValue;
    const int hc = height - 10, wc = width - 10;
    dim3 gf((wc + LT - 1) / LT, (hc + LT - 1) / LT);
    const size_t nf = gf.x * gf.y;
    if (!workspace) {
        *ws_bytes = al(8 * nf);
        return 0;
    }
    if (*ws_bytes < al(8 * nf)) return (int)cudaErrorInvalidValue;
    cudaStream_t s = (cudaStream_t)stream;
    double *pf = (double *)workspace;
    loss_smem_optin<double, double, double>();
    dim3 grid((wc + FW - 1) / FW, gf.y);
    ssim_fields_kernel<double, double, double><<<grid, LTHREADS, fields_smem<double>(), s>>>(
        height, width, channels, image, 0, ref, nullptr, 0, 0, 0, 0, height, pf);
    ISG_CHECK_LAUNCH();
    loss_finish_kernel<<<1, FINISH_THREADS, 0, s>>>((int)nf, pf, 0, nullptr, 0.0,
                                         (double)channels * hc * wc, 0.0, out_dev);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" const char *isg_version(void) {
    return "libisogs 0.2 sm_100a (preprocess fp64/glibc-exp, raster f32|f64, ssim f32|f64, "
           "row-band data plane)";
}
