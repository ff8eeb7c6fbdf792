// raster_common.cuh -- the float32 staged-entry form and the exact
// conservative box test shared by the rasteriser (raster_f32.cu) and the
// training path's live-tile binning (binning.cu).
#pragma once
#include "common.cuh"

namespace isg {
namespace f32 {

constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ float ex2a(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float lg2a(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Staged entry: g = (mx, my, -a/2, -b), h = (-c/2, thr, opacity, 0),
// c = (r, g, b, 0).  The scalings are exact (powers of two / sign).  box_dead
// reads this form; the inner loops read the base-2 form of to_log2().
struct Staged {
    float4 g, h, c;
};

// Exponent threshold below which opacity * exp(power) < 1/255 for certain:
// -ln(255 o) minus a margin far above the ex2/lg2 approximation error.
__device__ __forceinline__ float skip_thr(float op) {
    if (!(op > 0.0f)) return 1.0f;
    return __fsub_rn(__fmul_rn(lg2a(__fmul_rn(255.0f, op)), -LN2), 1e-3f);
}

__device__ __forceinline__ Staged stage(const float *__restrict__ feat, int rank) {
    const float4 *f = reinterpret_cast<const float4 *>(feat) + 3 * (int64_t)rank;
    const float4 x = __ldg(f), y = __ldg(f + 1), z = __ldg(f + 2);
    // x = (mx, my, a, b), y = (c, op, r, g), z = (b_col, 0, 0, 0)
    Staged s;
    s.g = make_float4(x.x, x.y, -0.5f * x.z, -x.w);
    s.h = make_float4(-0.5f * y.x, skip_thr(y.y), y.y, 0.0f);
    s.c = make_float4(y.z, y.w, z.x, 0.0f);
    return s;
}

// True when no pixel centre of the box [x0, x0+edge] x [y0, y0+edge] can
// reach the skip threshold: the exact maximum exponent over the box (convex
// quadratic: interior minimum or an edge minimum) is below thr by a margin
// that bounds the float rounding of the per-pixel exponent.
__device__ __forceinline__ bool box_dead(const Staged &s, float x0, float y0, float ex,
                                         float ey) {
    const float thr = s.h.y;
    if (thr > 0.0f) return true;  // opacity < 1/255: every pair is skipped
    const float a = -2.0f * s.g.z, b = -s.g.w, c = -2.0f * s.h.x;
    const float lx = x0 - s.g.x, hx = lx + ex, ly = y0 - s.g.y, hy = ly + ey;
    if (lx <= 0.0f && hx >= 0.0f && ly <= 0.0f && hy >= 0.0f) return false;
    float q = __int_as_float(0x7f800000);
#pragma unroll
    for (int e = 0; e < 2; e++) {
        const float d0 = e ? hx : lx;
        const float d1 = fminf(fmaxf(-b * d0 / c, ly), hy);
        q = fminf(q, a * d0 * d0 + 2.0f * b * d0 * d1 + c * d1 * d1);
        const float e1 = e ? hy : ly;
        const float e0 = fminf(fmaxf(-b * e1 / a, lx), hx);
        q = fminf(q, a * e0 * e0 + 2.0f * b * e0 * e1 + c * e1 * e1);
    }
    const float mdx = fmaxf(fabsf(lx), fabsf(hx)), mdy = fmaxf(fabsf(ly), fabsf(hy));
    const float scale = a * mdx * mdx + 2.0f * fabsf(b) * mdx * mdy + c * mdy * mdy;
    return -0.5f * q < thr - (1e-3f + 1e-5f * scale);
}

__device__ __forceinline__ bool box_dead(const Staged &s, float x0, float y0, float edge) {
    return box_dead(s, x0, y0, edge, edge);
}

// box_dead with the edge-minimiser slopes -b/c and -b/a precomputed once per
// splat (for many boxes of one splat: the training binning's tile test).  The
// clamped point differs from box_dead's by rounding only, and q there is still
// an upper bound of the box minimum whose error is second order (the point is
// a stationary point along the edge), far inside the margin: conservative.
struct CullForm {
    float4 p;  // (mx, my, a, b)
    float4 q;  // (c, thr, -b/c, -b/a)
};

__device__ __forceinline__ CullForm cull_form(const Staged &s) {
    const float a = -2.0f * s.g.z, b = -s.g.w, c = -2.0f * s.h.x;
    CullForm f;
    f.p = make_float4(s.g.x, s.g.y, a, b);
    f.q = make_float4(c, s.h.y, -b / c, -b / a);
    return f;
}

__device__ __forceinline__ bool box_dead_cf(const CullForm &f, float x0, float y0, float edge) {
    const float thr = f.q.y;
    if (thr > 0.0f) return true;
    const float a = f.p.z, b = f.p.w, c = f.q.x;
    const float lx = x0 - f.p.x, hx = lx + edge, ly = y0 - f.p.y, hy = ly + edge;
    if (lx <= 0.0f && hx >= 0.0f && ly <= 0.0f && hy >= 0.0f) return false;
    float q = __int_as_float(0x7f800000);
#pragma unroll
    for (int e = 0; e < 2; e++) {
        const float d0 = e ? hx : lx;
        const float d1 = fminf(fmaxf(f.q.z * d0, ly), hy);
        q = fminf(q, a * d0 * d0 + 2.0f * b * d0 * d1 + c * d1 * d1);
        const float e1 = e ? hy : ly;
        const float e0 = fminf(fmaxf(f.q.w * e1, lx), hx);
        q = fminf(q, a * e0 * e0 + 2.0f * b * e0 * e1 + c * e1 * e1);
    }
    const float mdx = fmaxf(fabsf(lx), fabsf(hx)), mdy = fmaxf(fabsf(ly), fabsf(hy));
    const float scale = a * mdx * mdx + 2.0f * fabsf(b) * mdx * mdy + c * mdy * mdy;
    return -0.5f * q < thr - (1e-3f + 1e-5f * scale);
}

}  // namespace f32
}  // namespace isg
