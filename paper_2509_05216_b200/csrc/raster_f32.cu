// raster_f32.cu -- production float32 tile rasteriser (sm_100a).
//
// _forward_tiles / _backward_tiles (_kernels.py:229-374) re-designed for the
// B200 SM.  Forward: one 128-thread CTA per 16x16 tile, warp w owns 8x8
// quadrant w, two pixels per lane (rows r and r+4 of one column, so the x
// terms of the exponent are shared).  Each warp stages 32 list entries at a
// time and keeps those its quadrant can see -- the exact maximum of the
// Gaussian exponent over the quadrant's pixel-centre box against the skip
// threshold (box_dead, raster_common.cuh; the margin covers the per-pixel
// rounding, so dropping an entry changes no result) -- then composites two
// entries per step with the decisions as predicates.  The training launch also
// leaves per-(tile, quadrant, batch) contribution masks for the backward.
//
// All decisions (skip, 0.99 clamp, stop) come from pair_alpha / pair_alpha_bl,
// written with explicit rounding intrinsics so the forward and the backward
// compute bit-identical exponents and alphas and therefore the same
// contributor sets.
//
// Backward: one 64-thread CTA per tile, warp h owns 16x8 half h, four pixels
// per lane; contributors walked back to front (T recovered by division from
// T_final).  Each pixel's exponent and alpha are computed unconditionally and
// a single branch on the forward's exact decision guards its gradient update
// (an early exit on the exponent would nest a second divergent branch per
// pixel, whose reconvergence costs more than the exp it saves).  The 9
// gradient terms of an entry are reduced over the warp with a
// butterfly reduce-scatter; the last warp to finish a batch folds both halves'
// sums in fixed order into the entry's (tile, splat) subtotal.  Deterministic
// throughout, no atomics on the data path.
#include "common.cuh"
#include "raster_f32.cuh"
#include "raster_common.cuh"

namespace isg {
namespace f32 {

constexpr int NT = 128;  // threads per tile (2 pixels each)
constexpr int NW = NT / 32;
constexpr int PSTRIDE = partial_stride<float>();  // floats per subtotal record
#ifndef BWD_MINB
#define BWD_MINB 12
#endif
// The quadratic-form coefficients and the threshold in base-2 units
// (multiplied by log2 e once per staged entry), so a pair's exponent feeds
// ex2 directly: power2 = log2(e) * power.
__device__ __forceinline__ void to_log2(Staged &s) {
    s.g.z = __fmul_rn(s.g.z, LOG2E);
    s.g.w = __fmul_rn(s.g.w, LOG2E);
    s.h.x = __fmul_rn(s.h.x, LOG2E);
    s.h.y = __fmul_rn(s.h.y, LOG2E);
}

// Column terms of the exponent shared by a thread's two pixels (same x):
// power2 = A + d1 * (B + nc * d1) with A = na d0^2, B = nb d0 (base 2).
__device__ __forceinline__ void col_terms(float d0, const float4 &g4, float &A, float &B) {
    A = __fmul_rn(__fmul_rn(g4.z, d0), d0);
    B = __fmul_rn(g4.w, d0);
}

// Per-pair alpha (0 when the pair is skipped) and the unclamped product
// o * g.  The threshold test is an early exit only: a pair below it also
// fails alpha >= 1/255 (the margin dominates the ex2/lg2 error), so
// pair_alpha and pair_alpha_bl make identical decisions.
__device__ __forceinline__ float pair_alpha(float d1, float A, float B, const float4 &h4,
                                            float &og) {
    const float power = __fmaf_rn(d1, __fmaf_rn(h4.x, d1, B), A);
    if (power > 0.0f || power < h4.y) return 0.0f;
    og = __fmul_rn(h4.z, ex2a(power));
    const float a = fminf(og, 0.99f);
    return a >= (1.0f / 255.0f) ? a : 0.0f;
}

// pair_alpha without the early exit (ex2 always evaluated): the same bits for
// every pair, so several pairs' alphas can be computed ahead of the
// sequential compositing.  Returns the clamped alpha; `on` = the pair is
// composited unless the pixel stops (the same decision as pair_alpha > 0).
__device__ __forceinline__ float pair_alpha_bl(float d1, float A, float B, const float4 &h4,
                                               bool &on) {
    const float power = __fmaf_rn(d1, __fmaf_rn(h4.x, d1, B), A);
    const float a = fminf(__fmul_rn(h4.z, ex2a(power)), 0.99f);
    on = !(power > 0.0f) && a >= (1.0f / 255.0f);
    return a;
}

// Packed float32 pairs (fma/add/mul.rn.ftz.f32x2: FFMA2 / FADD2 / FMUL2, two
// lanes' worth of IEEE operations per issue slot, each component bitwise the
// scalar instruction).  A thread's pixels of one column share an entry's
// coefficients, which the SM reads as broadcast (.F32) operands: the
// exponent of two pixels costs three packed instructions instead of six.
// Measured at config 3: backward 3.50 -> 3.465 ms, forward 1.877 -> 1.873 ms,
// losses bitwise unchanged.
#ifndef FWD_PACK2
#define FWD_PACK2 1
#endif
#ifndef BWD_PACK2
#define BWD_PACK2 1
#endif
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t pk2(float a, float b) {
    f2_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void up2(f2_t r, float &a, float &b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c) {
    f2_t r;
    asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ f2_t add2(f2_t a, f2_t b) {
    f2_t r;
    asm("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2_t mul2(f2_t a, f2_t b) {
    f2_t r;
    asm("mul.rn.ftz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
// pair_alpha_bl for a thread's two pixels at rows y0, y1 (same column):
// the same bits per pixel.  d1 is returned for the backward's gradient.
__device__ __forceinline__ void pair_alpha_bl2(float y0, float y1, float gy, float A, float B,
                                               const float4 &h4, float &p0, float &p1,
                                               float &og0, float &og1, float &d10, float &d11) {
    const f2_t d = add2(pk2(y0, y1), pk2(-gy, -gy));
    const f2_t pw = fma2(d, fma2(pk2(h4.x, h4.x), d, pk2(B, B)), pk2(A, A));
    up2(pw, p0, p1);
    up2(d, d10, d11);
    const f2_t og = mul2(pk2(h4.z, h4.z), pk2(ex2a(p0), ex2a(p1)));
    up2(og, og0, og1);
}

// Reachability mask of one staged entry over the four 8x8 quadrants of the
// tile (bit q = quadrant (q & 1, q >> 1)); 0 when the whole tile is dead.
__device__ __forceinline__ unsigned quad_mask(const Staged &st, float x0, float y0) {
    if (box_dead(st, x0, y0, 15.0f)) return 0u;
    unsigned m = 0u;
#pragma unroll
    for (int q = 0; q < 4; q++)
        if (!box_dead(st, x0 + 8.0f * (q & 1), y0 + 8.0f * (q >> 1), 7.0f)) m |= 1u << q;
    return m;
}

// ------------------------------------------------------------- forward ----
// Shared-memory accessors on 32-bit shared-window addresses, so the inner
// loops carry one base register per array instead of re-deriving generic
// addresses every iteration.
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    // opaque copy: keeps the address in a register instead of letting the
    // compiler re-derive the shared window base at every use
    uint32_t r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return r;
}
__device__ __forceinline__ float4 lds4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts(uint32_t a, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ int ldsu8(uint32_t a) {
    unsigned short v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(a));
    return (int)v;
}

// Backward work items: a tile's list is cut into chunks of `chunk` entries
// (a multiple of WB; 0 = one chunk per tile) that run as separate CTAs; the
// forward leaves, per pixel, (T, r, g, b) before every internal chunk
// boundary at cstate[256 * chunk_slot + pixel].  Slots are unique per
// (tile, boundary): e0 / chunk + tl + k <= E / chunk + n_tiles.
constexpr int LAST_CHUNK = 1 << 30;  // item flag: the chunk runs to the list end
__device__ __forceinline__ int64_t chunk_slot(int e0, int tl, int base, int chunk) {
    return (int64_t)(e0 / chunk) + tl + base / chunk;
}

// Forward kernel modes: TOUCH counts per-splat touches (the reference's
// `touched`), STATS records n_contrib / n_iter (bench statistics only).
constexpr int F_TOUCH = 1, F_STATS = 2;
#define FINF __int_as_float(0x7f800000)

// Front-to-back compositing of one pair (_kernels.py:258-272): skipped when
// alpha is 0; stops (without compositing) when T would drop below 1e-4.  A
// finished pixel moves its row coordinate to +inf, so every later exponent is
// -inf and every later alpha 0 (c > 0 for every staged conic): no done flag is
// carried.  CHECK re-tests that sentinel for an alpha computed before the
// pixel finished (the second entry of a step).
template <int MODE, bool CHECK>
__device__ __forceinline__ bool composite(float a, bool on, int slot, int base, uint32_t a_col,
                                          float &fpy, int &it, float &t, float &r, float &g,
                                          float &b, int &last, int &cnt, unsigned &cm) {
    if (!on || (CHECK && fpy == FINF)) return false;
    const float test = t * (1.0f - a);
    if (test < 1e-4f) {
        fpy = FINF;
        if (MODE & F_STATS) it = base + slot + 1;
        return false;
    }
    const float4 c = lds4(a_col + 16 * slot);
    const float w = a * t;
    r = fmaf(c.x, w, r);
    g = fmaf(c.y, w, g);
    b = fmaf(c.z, w, b);
    t = test;
    last = base + slot + 1;
    cm |= 1u << slot;
    if (MODE & F_STATS) cnt++;
    return true;
}

// Touch counts (the reference's `touched`): the pixels of the warp's quadrant
// that composited a slot, added with one atomic per (quadrant, entry).
__device__ __forceinline__ void touch_add(bool c0, bool c1, int slot, int64_t *touched,
                                          const int *srank) {
    const unsigned n = __popc(__ballot_sync(FULL, c0)) + __popc(__ballot_sync(FULL, c1));
    if (n && (threadIdx.x & 31) == 0)
        atomicAdd((unsigned long long *)&touched[srank[slot]], (unsigned long long)n);
}

// composite() for the training launch (no touch / stats counters), written so
// the decisions are predicates and the updates predicated moves and FMAs
// (the SM's ALU pipe, which carries compares and selects, is the forward's
// busiest): the same decisions and the same bits.  jn = the entry's list
// index + 1.  Returns whether the pair was composited.
template <bool CHECK>
__device__ __forceinline__ bool composite_pr(float a, bool on, const float4 &c, int jn,
                                             float &fpy, float &t, float &r, float &g, float &b,
                                             int &last) {
    if (CHECK) on = on && fpy != FINF;
    const float test = t * (1.0f - a);
    const bool stop = test < 1e-4f;
    const bool comp = on && !stop;
    if (comp) {
        const float w = a * t;
        r = fmaf(c.x, w, r);
        g = fmaf(c.y, w, g);
        b = fmaf(c.z, w, b);
        t = test;
        last = jn;
    }
    if (on && stop) fpy = FINF;
    return comp;
}

// Warp w renders quadrant (w & 1, w >> 1) of the tile: lane (lx, ly) owns
// pixels (lx, ly) and (lx, ly + 4) of the 8x8 quadrant.  The four warps run
// independently (no block barrier): each walks the tile's entry list in
// batches of 32, stages one entry per lane in its own shared slice, keeps the
// entries that can reach its quadrant (box_dead over the 8x8 pixel box) and
// composites them.  "All pixels done" is tested every FCHK entries (a
// finished pixel only skips work, so the late test changes no result).
#ifndef FWD_FCHK
#define FWD_FCHK 32
#endif
constexpr int FCHK = FWD_FCHK;
constexpr int WB = 32;  // per-warp staging batch

#ifndef FWD_MINB
#define FWD_MINB 6
#endif
template <int MODE>
__global__ void __launch_bounds__(NT, FWD_MINB) fwd_kernel(
    int W, int H, int tiles_x, int row_lo, const int32_t *__restrict__ tile_ids,
    const int32_t *__restrict__ tile_order, const int32_t *__restrict__ offsets,
    const int32_t *__restrict__ entries, const float *__restrict__ feat, float bg0, float bg1,
    float bg2, void *image, int image_f64,
    float *__restrict__ t_final, int32_t *__restrict__ n_last, int32_t *__restrict__ n_contrib,
    int32_t *__restrict__ n_iter, int64_t *__restrict__ touched, uint32_t *__restrict__ cmask,
    int chunk, float4 *__restrict__ cstate, int32_t *__restrict__ qlast,
    const int32_t *__restrict__ slot_rank) {
    constexpr bool TOUCH = MODE & F_TOUCH;
    // slot WB of each warp's slice is a sentinel entry that never composites
    // (opacity 0): odd lists are padded with it, so entries go two at a time
    __shared__ float4 sgh_all[NW][WB + 1][2];
    __shared__ float4 scol_all[NW][WB + 1];
    __shared__ int srank_all[NW][TOUCH ? WB : 1];
    __shared__ unsigned char slist_all[NW][WB + 1];
    const int tl = tile_order ? tile_order[blockIdx.x] : blockIdx.x;
    const int tid = tile_ids ? tile_ids[tl] : row_lo * tiles_x + tl;
    const int ty = tid / tiles_x, tx = tid - ty * tiles_x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int px = tx * 16 + (warp & 1) * 8 + (lane & 7);
    const int py0 = ty * 16 + (warp >> 1) * 8 + (lane >> 3), py1 = py0 + 4;
    const bool in0 = px < W && py0 < H, in1 = px < W && py1 < H;
    const float fpx = (float)px;
    float fpy0 = in0 ? (float)py0 : FINF, fpy1 = in1 ? (float)py1 : FINF;
    const float qx0 = (float)(tx * 16 + (warp & 1) * 8), qy0 = (float)(ty * 16 + (warp >> 1) * 8);
    const int e0 = offsets[tl], n_ent = offsets[tl + 1] - e0;
    float4(&sgh)[WB + 1][2] = sgh_all[warp];
    float4(&scol)[WB + 1] = scol_all[warp];
    int *srank = srank_all[warp];
    if (lane == 0) {
        const float4 z = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        sgh[WB][0] = z;
        sgh[WB][1] = z;  // power 0, opacity 0: alpha 0 at every pixel
        scol[WB] = z;
    }
    const uint32_t a_gh = smem_addr(&sgh[0][0]), a_col = smem_addr(&scol[0]);
    const uint32_t a_list = smem_addr(&slist_all[warp][0]);
    const unsigned lt = (1u << lane) - 1u;
    float t0 = 1.0f, r0 = 0.0f, g0 = 0.0f, b0 = 0.0f;
    float t1 = 1.0f, r1 = 0.0f, g1 = 0.0f, b1 = 0.0f;
    int last0 = 0, last1 = 0, cnt0 = 0, cnt1 = 0, it0 = 0, it1 = 0;
    for (int base = 0; base < n_ent; base += WB) {
        if (__all_sync(FULL, fpy0 == FINF && fpy1 == FINF)) break;
        if (cstate && base > 0 && base % chunk == 0) {
            // state before entry `base` for the backward's chunk ending there
            // (a warp with every pixel done has left the loop: the backward
            // never reads a boundary past a pixel's last contributor)
            float4 *cs = cstate + 256 * chunk_slot(e0, tl, base, chunk);
            const int c = (warp & 1) * 8 + (lane & 7), r = (warp >> 1) * 8 + (lane >> 3);
            cs[16 * r + c] = make_float4(t0, r0, g0, b0);
            cs[16 * (r + 4) + c] = make_float4(t1, r1, g1, b1);
        }
        const int j = base + lane;
        bool alive = false;
        if (j < n_ent) {
            // live-only lists hold subtotal slots: slot_rank maps them to ranks
            const int32_t ent = entries[e0 + j];
            const int rank = slot_rank ? slot_rank[ent] : ent;
            Staged st = stage(feat, rank);
            alive = !box_dead(st, qx0, qy0, 7.0f);
            to_log2(st);
            sgh[lane][0] = st.g;
            sgh[lane][1] = st.h;
            scol[lane] = st.c;
            if (TOUCH) srank[lane] = rank;
        }
        const unsigned bal = __ballot_sync(FULL, alive);
        if (alive) slist_all[warp][__popc(bal & lt)] = (unsigned char)lane;
        const int total = __popc(bal);
        if (lane == 0) slist_all[warp][total] = (unsigned char)WB;  // odd-length pad
        __syncwarp();
        unsigned cm = 0u;  // batch slots this lane's pixels composited
        for (int k0 = 0; k0 < total; k0 += FCHK) {
            if (k0 && __all_sync(FULL, fpy0 == FINF && fpy1 == FINF)) break;
            const int kend = min(k0 + FCHK, total);
            // two entries per step: the four pair alphas are independent and
            // computed ahead; compositing stays in list order per pixel
            for (int k = k0; k < kend; k += 2) {
                // slot WB (the sentinel) when k + 1 == total
                const int sa = ldsu8(a_list + k), sb = ldsu8(a_list + k + 1);
                const float4 ga = lds4(a_gh + 32 * sa), ha = lds4(a_gh + 32 * sa + 16);
                const float4 gb = lds4(a_gh + 32 * sb), hb = lds4(a_gh + 32 * sb + 16);
                float Aa, Ba, Ab, Bb;
                col_terms(fpx - ga.x, ga, Aa, Ba);
                col_terms(fpx - gb.x, gb, Ab, Bb);
                bool oa0, oa1, ob0, ob1;
#if FWD_PACK2
                float aa0, aa1, ab0, ab1;
                {
                    float p0, p1, q0, q1, o0, o1, u0, u1, dd0, dd1;
                    pair_alpha_bl2(fpy0, fpy1, ga.y, Aa, Ba, ha, p0, p1, o0, o1, dd0, dd1);
                    pair_alpha_bl2(fpy0, fpy1, gb.y, Ab, Bb, hb, q0, q1, u0, u1, dd0, dd1);
                    aa0 = fminf(o0, 0.99f);
                    aa1 = fminf(o1, 0.99f);
                    ab0 = fminf(u0, 0.99f);
                    ab1 = fminf(u1, 0.99f);
                    oa0 = !(p0 > 0.0f) && aa0 >= (1.0f / 255.0f);
                    oa1 = !(p1 > 0.0f) && aa1 >= (1.0f / 255.0f);
                    ob0 = !(q0 > 0.0f) && ab0 >= (1.0f / 255.0f);
                    ob1 = !(q1 > 0.0f) && ab1 >= (1.0f / 255.0f);
                }
#else
                const float aa0 = pair_alpha_bl(fpy0 - ga.y, Aa, Ba, ha, oa0);
                const float aa1 = pair_alpha_bl(fpy1 - ga.y, Aa, Ba, ha, oa1);
                const float ab0 = pair_alpha_bl(fpy0 - gb.y, Ab, Bb, hb, ob0);
                const float ab1 = pair_alpha_bl(fpy1 - gb.y, Ab, Bb, hb, ob1);
#endif
                if (MODE == 0) {
                    const float4 ca = lds4(a_col + 16 * sa), cb = lds4(a_col + 16 * sb);
                    const int ja = base + sa + 1, jb = base + sb + 1;
                    const bool ca0 = composite_pr<false>(aa0, oa0, ca, ja, fpy0, t0, r0, g0, b0, last0);
                    const bool ca1 = composite_pr<false>(aa1, oa1, ca, ja, fpy1, t1, r1, g1, b1, last1);
                    const bool cb0 = composite_pr<true>(ab0, ob0, cb, jb, fpy0, t0, r0, g0, b0, last0);
                    const bool cb1 = composite_pr<true>(ab1, ob1, cb, jb, fpy1, t1, r1, g1, b1, last1);
                    if (ca0 || ca1) cm |= 1u << sa;
                    if (cb0 || cb1) cm |= 1u << sb;
                } else {
                    const bool ca0 = composite<MODE, false>(aa0, oa0, sa, base, a_col, fpy0, it0,
                                                            t0, r0, g0, b0, last0, cnt0, cm);
                    const bool ca1 = composite<MODE, false>(aa1, oa1, sa, base, a_col, fpy1, it1,
                                                            t1, r1, g1, b1, last1, cnt1, cm);
                    const bool cb0 = composite<MODE, true>(ab0, ob0, sb, base, a_col, fpy0, it0,
                                                           t0, r0, g0, b0, last0, cnt0, cm);
                    const bool cb1 = composite<MODE, true>(ab1, ob1, sb, base, a_col, fpy1, it1,
                                                           t1, r1, g1, b1, last1, cnt1, cm);
                    if (TOUCH) {
                        touch_add(ca0, ca1, sa, touched, srank);
                        touch_add(cb0, cb1, sb, touched, srank);
                    }
                }
            }
        }
        // contribution mask of this (tile, quadrant, batch) for the backward:
        // bit s = batch slot s was composited by some pixel of the quadrant
        if (cmask) {
            cm = __reduce_or_sync(FULL, cm);
            if (lane == 0) cmask[4 * ((int64_t)(e0 >> 5) + tl + (base >> 5)) + warp] = cm;
        }
        __syncwarp();  // the slice is restaged next batch
    }
    if (qlast) {
        // the quadrant's last composited list position: the backward cuts
        // chunks only below it (past it every entry's subtotal is zero)
        int ql = max(last0, last1);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ql = max(ql, __shfl_xor_sync(FULL, ql, o));
        if (lane == 0) qlast[4 * tl + warp] = ql;
    }
#pragma unroll
    for (int p = 0; p < 2; p++) {
        const bool in = p ? in1 : in0;
        if (!in) continue;
        const int py = p ? py1 : py0;
        const float t = p ? t1 : t0;
        const int64_t pix = (int64_t)py * W + px;
        const float vr = fmaf(t, bg0, p ? r1 : r0), vg = fmaf(t, bg1, p ? g1 : g0),
                    vb = fmaf(t, bg2, p ? b1 : b0);
        if (image_f64) {
            double *im = (double *)image + 3 * pix;
            im[0] = vr;
            im[1] = vg;
            im[2] = vb;
        } else {
            float *im = (float *)image + 3 * pix;
            im[0] = vr;
            im[1] = vg;
            im[2] = vb;
        }
        t_final[pix] = t;
        n_last[pix] = p ? last1 : last0;
        if (MODE & F_STATS) {
            if (n_contrib) n_contrib[pix] = p ? cnt1 : cnt0;
            if (n_iter) n_iter[pix] = (p ? fpy1 : fpy0) == FINF ? (p ? it1 : it0) : n_ent;
        }
    }
}

// ------------------------------------------------------------ backward ----
// Butterfly reduce-scatter of 9 values over the warp (12 shuffles).  After it,
// lane L with bits (b4,b3,b2,b1) holds the full sum of value
// 5*b4 + 3*b3 + 2*b2 + b1 (see bfly_slot).
__device__ __forceinline__ float bfly9(const float (&v)[9], int lane) {
    // Each level keeps one of a pair of value columns per lane and adds the
    // partner's copy of the same column.  Where the pair's second column is
    // padding (past the 9 values), every lane simply adds the partner's first
    // column: the lanes that "keep" the padding then hold a duplicate in a
    // padding column, which never reaches a valid slot (columns are summed
    // independently) -- two selects fewer per padded pair.
    const bool s4 = lane & 16, s3 = lane & 8, s2 = lane & 4, s1 = lane & 2;
    float u[5];
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const float a = v[i], b = v[i + 5];
        u[i] = (s4 ? b : a) + __shfl_xor_sync(FULL, s4 ? a : b, 16);
    }
    u[4] = v[4] + __shfl_xor_sync(FULL, v[4], 16);
    float w[3];
#pragma unroll
    for (int i = 0; i < 2; i++) {
        const float a = u[i], b = u[i + 3];
        w[i] = (s3 ? b : a) + __shfl_xor_sync(FULL, s3 ? a : b, 8);
    }
    w[2] = u[2] + __shfl_xor_sync(FULL, u[2], 8);
    float x[2];
    x[0] = (s2 ? w[2] : w[0]) + __shfl_xor_sync(FULL, s2 ? w[0] : w[2], 4);
    x[1] = w[1] + __shfl_xor_sync(FULL, w[1], 4);
    float y = (s1 ? x[1] : x[0]) + __shfl_xor_sync(FULL, s1 ? x[0] : x[1], 2);
    return y + __shfl_xor_sync(FULL, y, 1);
}

// Value index held by `lane` after bfly9, or -1 (pad / duplicate lane).
__device__ __forceinline__ int bfly_slot(int lane) {
    if (lane & 1) return -1;
    const int b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1, b2 = (lane >> 2) & 1, b1 = (lane >> 1) & 1;
    const int f = 5 * b4 + 3 * b3 + 2 * b2 + b1;
    return ((2 * b2 + b1) < (b3 ? 2 : 3) && f < 9) ? f : -1;
}

// One contributing (pixel, entry) pair: accumulate its 9 gradient terms and
// advance the pixel's back-to-front state (T, S).  _kernels.py:342-374.
__device__ __forceinline__ float rcpa(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Per-entry quantities shared by a thread's pixels (same column).
// Per pixel the backward keeps T and Q = sum_c dL/dC_c * S_c (the reference's
// three running sums S_c only ever enter dalpha through this dot product), so
//   dalpha = wc * T_before - Q / (1 - alpha),  Q += wc * alpha * T_before,
// with wc = sum_c dL/dC_c * colour_c.  The conic and mean terms are moments
// of dpower = dalpha * o * g over the thread's pixels (s0 = sum dp,
// s1 = sum dp d1, s2 = sum dp d1^2; d0 is shared), turned into linear moments
// by moment_terms; s0 also carries the opacity term (dopacity = sum dalpha g
// = s0 / o, divided once per (tile, entry) in the fold).
#ifndef BWD_FLAT_CLAMP
#define BWD_FLAT_CLAMP 0
#endif
__device__ __forceinline__ void pair_grad(float a, float og, float d1, float wc, float wr,
                                          float wg, float wb, float &T, float &Q, float (&v)[9],
                                          float &s0, float &s1, float &s2) {
    const float inv = rcpa(1.0f - a);
    const float ti = T * inv;  // T before this splat
    const float at = a * ti;
    v[5] = fmaf(wr, at, v[5]);
    v[6] = fmaf(wg, at, v[6]);
    v[7] = fmaf(wb, at, v[7]);
    const float dalpha = fmaf(wc, ti, -(Q * inv));
    Q = fmaf(wc, at, Q);
#if BWD_FLAT_CLAMP
    // clamped alpha: zero sub-gradient, as a select instead of a branch
    const float dp = og > 0.99f ? 0.0f : dalpha * og;
    const float t = dp * d1;
    s0 += dp;
    s1 += t;
    s2 = fmaf(t, d1, s2);
#else
    if (!(og > 0.99f)) {  // clamped alpha: zero sub-gradient
        const float dp = dalpha * og;
        const float t = dp * d1;
        s0 += dp;
        s1 += t;
        s2 = fmaf(t, d1, s2);
    }
#endif
    T = ti;
}

// The conic and mean terms leave the warp as linear moments (summed over
// lanes and quadrants like every other term):
//   v0 = sum d0 dp, v1 = sum dp d1, v2 = sum d0^2 dp, v3 = sum d0 dp d1,
//   v4 = sum dp d1^2
// and are expanded once per (tile, entry) in the fold (_kernels.py:363-374):
//   dmean = (a v0 + b v1, b v0 + c v1), dconic = (-v2/2, -v3, -v4/2).
__device__ __forceinline__ void moment_terms(float d0, float s0, float s1, float s2,
                                             float (&v)[9]) {
    v[8] = s0;
    const float d0s0 = d0 * s0;
    v[0] = d0s0;
    v[1] = s1;
    v[2] = d0 * d0s0;
    v[3] = d0 * s1;
    v[4] = s2;
}

// Backward: one 64-thread CTA per tile, one warp per 16x8 half (four pixels
// per thread: column lane & 15, rows (lane >> 4) + {0, 2, 4, 6}), so the
// 9-value butterfly per entry is amortised over 128 pixels; the coarser cull
// box costs fewer instructions than the halved reductions save.  The two
// warps run independently.  Each walks the tile's entry list back to front in
// batches of WB, stages the batch in its own shared slice, keeps the entries
// that reach its half (and lie before its last contributor) and leaves one
// 9-value warp sum per kept entry in a ring of RING batch slots.  The last
// warp to finish a batch (shared-memory arrival counter) folds it: per entry,
// the halves that kept it in fixed order, then the moment expansion, one
// padded record per (tile, entry).  A warp may run up to RING-1 batches ahead
// of the other; it waits only when its ring slot has not been folded yet.
#ifndef BWD_RING
#define BWD_RING 3
#endif
#ifndef BWD_FLAT_ALPHA
#define BWD_FLAT_ALPHA 1
#endif
constexpr int RING = BWD_RING;

#ifndef BWD_SLEEP
#define BWD_SLEEP 256
#endif
__device__ __forceinline__ int ld_volatile(const int *p) {
    return *reinterpret_cast<const volatile int *>(p);
}

constexpr int BNT = 64;  // backward threads per tile (two 16x8 halves)

// UNR > 1: the entry loop takes UNR entries per step (their exponents and
// butterflies are independent, so a warp that runs alone on its SM -- the tail
// of a one-wave launch -- has UNR times the instruction-level parallelism);
// every pixel still walks its entries in list order, so the results are the
// bits of UNR = 1.  Measured on emulated W = 8 bands (config 3): UNR 2 491,
// 3 496, 4 474 images/s.
#ifndef BWD_UNR
#define BWD_UNR 3
#endif
#ifndef BWD_MINB2
#define BWD_MINB2 1
#endif
template <typename DL, bool MASK, bool CHUNKED, int UNR = 1>
__global__ void __launch_bounds__(BNT, UNR == 1 ? BWD_MINB : BWD_MINB2) bwd_kernel(
    int W, int H, int tiles_x, int row_lo, const int32_t *__restrict__ tile_ids,
    const int32_t *__restrict__ tile_order, const int32_t *__restrict__ offsets,
    const int32_t *__restrict__ entries, const float *__restrict__ feat,
    const int4 *__restrict__ rect_sorted,
    const int64_t *__restrict__ emit_off, float bg0, float bg1, float bg2,
    const float *__restrict__ t_final, const int32_t *__restrict__ n_last,
    const DL *__restrict__ dl, float *__restrict__ partials, const uint32_t *__restrict__ cmask,
    const int2 *__restrict__ items, const int32_t *__restrict__ n_items, int chunk,
    const float4 *__restrict__ cstate, const float *__restrict__ image,
    const int32_t *__restrict__ slot_rank) {
    constexpr int NH = BNT / 32;  // warps per tile: one per 16x8 half
    __shared__ float4 sgh_all[NH][WB][2];
    __shared__ float4 scol_all[NH][WB];
    __shared__ unsigned char slist_all[NH][WB];
    __shared__ float sred[RING][NH][WB][9];
    __shared__ unsigned spres[RING][NH];
    __shared__ int sarrive[RING];
    __shared__ int sfolded[RING];
    int tl, ck = 0;  // tile list position, chunk
    if (CHUNKED) {
        if ((int)blockIdx.x >= __ldg(n_items)) return;
        const int2 it = items[blockIdx.x];
        tl = it.x;
        ck = it.y;  // chunk index | LAST_CHUNK
    } else {
        tl = tile_order ? tile_order[blockIdx.x] : blockIdx.x;
    }
    const int tid = tile_ids ? tile_ids[tl] : row_lo * tiles_x + tl;
    const int ty = tid / tiles_x, tx = tid - ty * tiles_x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // lane (col, rg) owns column col and rows rg + {0, 2, 4, 6} of its half
    const int px = tx * 16 + (lane & 15);
    const int pyb = ty * 16 + warp * 8 + (lane >> 4);
    const float fpx = (float)px;
    const float qx0 = (float)(tx * 16), qy0 = (float)(ty * 16 + warp * 8);
    const int e0t = offsets[tl], n_ent = offsets[tl + 1] - e0t;
    // this item's entries [c_a, c_b) of the tile's list; the walk below is
    // relative to c_a (entries, list positions, contribution-mask words), so
    // the chunked and whole-tile instantiations run the same loop
    const int c_a = CHUNKED ? (ck & ~LAST_CHUNK) * chunk : 0;
    const int c_b = CHUNKED && !(ck & LAST_CHUNK) ? c_a + chunk : n_ent;
    const int e0 = e0t + c_a, n_item = c_b - c_a;
    const int64_t cm_base = 4 * ((int64_t)(e0t >> 5) + tl + (c_a >> 5)) + 2 * warp;
    const int my_slot = bfly_slot(lane);
    float4(&sgh)[WB][2] = sgh_all[warp];
    float4(&scol)[WB] = scol_all[warp];
    const uint32_t a_gh = smem_addr(&sgh[0][0]), a_col = smem_addr(&scol[0]);
    const uint32_t a_list = smem_addr(&slist_all[warp][0]);
    const unsigned lt = (1u << lane) - 1u;
    if (threadIdx.x < RING) {
        sarrive[threadIdx.x] = 0;
        sfolded[threadIdx.x] = (int)threadIdx.x - RING;  // slot r is free for batch r
    }

    int last[4];
    float T[4], Q[4], wr[4], wg[4], wb[4], fpy[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int py = pyb + 2 * q;
        fpy[q] = (float)py;
        last[q] = 0;
        T[q] = wr[q] = wg[q] = wb[q] = 0.0f;
        if (px < W && py < H) {
            const int64_t pix = (int64_t)py * W + px;
            last[q] = n_last[pix];
            T[q] = t_final[pix];
            wr[q] = (float)dl[3 * pix];
            wg[q] = (float)dl[3 * pix + 1];
            wb[q] = (float)dl[3 * pix + 2];
        }
        if (CHUNKED && last[q] > c_b) {
            // the pixel composited past this chunk: start from the forward's
            // state before entry c_b, with S = image - colour accumulated so far
            const float4 st = cstate[256 * chunk_slot(e0t, tl, c_b, chunk) +
                                     16 * (pyb + 2 * q - ty * 16) + (px - tx * 16)];
            const int64_t pix = (int64_t)(pyb + 2 * q) * W + px;
            T[q] = st.x;
            Q[q] = wr[q] * (image[3 * pix] - st.y) + wg[q] * (image[3 * pix + 1] - st.z) +
                   wb[q] * (image[3 * pix + 2] - st.w);
        } else {
            // Q = sum_c w_c S_c with S_c starting at T_final * bg_c
            Q[q] = wr[q] * (T[q] * bg0) + wg[q] * (T[q] * bg1) + wb[q] * (T[q] * bg2);
        }
        last[q] -= c_a;  // item-relative (<= 0: nothing of this item)
    }
    // nothing is composited at j >= wm; wq0 / wq1: the same bound over the
    // left / right 8x8 quadrant of this half (columns lane & 8)
    int wq = max(max(last[0], last[1]), max(last[2], last[3]));
    wq = max(wq, __shfl_xor_sync(FULL, wq, 16));
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) wq = max(wq, __shfl_xor_sync(FULL, wq, o));
    const int wq0 = __shfl_sync(FULL, wq, 0), wq1 = __shfl_sync(FULL, wq, 8);
    const int wm = max(wq0, wq1);
    __syncthreads();  // ring state initialised

    // batches of WB entries aligned at the list start (the forward's batches,
    // so the contribution masks line up), walked last to first
    const int n_b = (n_item + WB - 1) / WB;
    for (int bi = 0; bi < n_b; bi++) {
        const int start = (n_b - 1 - bi) * WB, end = min(start + WB, n_item);
        const int rs = bi % RING;
        if (lane == 0)
            while (ld_volatile(&sfolded[rs]) != bi - RING) __nanosleep(BWD_SLEEP);
        __syncwarp();
        const int j = start + lane;
        bool alive = false;
        if (MASK) {
            // the forward's contribution masks of the half's two quadrants:
            // exactly the entries some pixel of the half composited (a
            // quadrant's mask is valid while its forward warp was running)
            const int64_t w = cm_base + 4 * (start >> 5);
            unsigned bm = 0u;
            if (start < wq0) bm |= __ldg(cmask + w);
            if (start < wq1) bm |= __ldg(cmask + w + 1);
            alive = (bm >> lane) & 1u;
        }
        if (MASK ? alive : (j < end && j < wm)) {
            const int32_t ent = entries[e0 + j];
            Staged st = stage(feat, slot_rank ? slot_rank[ent] : ent);
            if (!MASK) alive = !box_dead(st, qx0, qy0, 15.0f, 7.0f);
            to_log2(st);
            sgh[lane][0] = st.g;
            sgh[lane][1] = st.h;
            scol[lane] = st.c;
        }
        const unsigned bal = __ballot_sync(FULL, alive);
        if (alive) slist_all[warp][__popc(bal & lt)] = (unsigned char)lane;
        __syncwarp();
        const uint32_t a_red = smem_addr(&sred[rs][warp][0][0]) + 4u * (uint32_t)max(my_slot, 0);
        int k = __popc(bal) - 1;
        if (UNR > 1) {
            for (; k >= UNR - 1; k -= UNR) {
                // entries sa (later in the list, walked first) and sb
                int sl[UNR];
#pragma unroll
                for (int e = 0; e < UNR; e++) sl[e] = ldsu8(a_list + k - e);
                float4 g4[UNR], h4[UNR], col[UNR];
                float d0[UNR], pw[UNR][4], ogv[UNR][4], dv[UNR][4];
#pragma unroll
                for (int e = 0; e < UNR; e++) {
                    const uint32_t ag = a_gh + 32 * sl[e];
                    g4[e] = lds4(ag);
                    h4[e] = lds4(ag + 16);
                    col[e] = lds4(a_col + 16 * sl[e]);
                    d0[e] = fpx - g4[e].x;
                    float A, B;
                    col_terms(d0[e], g4[e], A, B);
                    pair_alpha_bl2(fpy[0], fpy[1], g4[e].y, A, B, h4[e], pw[e][0], pw[e][1],
                                   ogv[e][0], ogv[e][1], dv[e][0], dv[e][1]);
                    pair_alpha_bl2(fpy[2], fpy[3], g4[e].y, A, B, h4[e], pw[e][2], pw[e][3],
                                   ogv[e][2], ogv[e][3], dv[e][2], dv[e][3]);
                }
                float v[UNR][9], sm[UNR][3];
#pragma unroll
                for (int e = 0; e < UNR; e++) {
#pragma unroll
                    for (int q = 0; q < 9; q++) v[e][q] = 0.0f;
                    sm[e][0] = sm[e][1] = sm[e][2] = 0.0f;
                    const int jj = start + sl[e];
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const float a = fminf(ogv[e][q], 0.99f);
                        if (jj < last[q] && !(pw[e][q] > 0.0f) && a >= (1.0f / 255.0f)) {
                            const float wc = fmaf(wb[q], col[e].z, fmaf(wg[q], col[e].y, wr[q] * col[e].x));
                            pair_grad(a, ogv[e][q], dv[e][q], wc, wr[q], wg[q], wb[q], T[q], Q[q],
                                      v[e], sm[e][0], sm[e][1], sm[e][2]);
                        }
                    }
                }
#pragma unroll
                for (int e = 0; e < UNR; e++) {
                    moment_terms(d0[e], sm[e][0], sm[e][1], sm[e][2], v[e]);
                    const float y = bfly9(v[e], lane);
                    if (my_slot >= 0) sts(a_red + 36u * (uint32_t)sl[e], y);
                }
            }
        }
        for (; k >= 0; k--) {
            const int slot = ldsu8(a_list + k);
            const uint32_t ag = a_gh + 32 * slot;
            const float4 g4 = lds4(ag), h4 = lds4(ag + 16);
            const int jj = start + slot;
            float v[9];
#pragma unroll
            for (int q = 0; q < 9; q++) v[q] = 0.0f;
            float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f;
            const float d0 = fpx - g4.x;
            float A, B;
            col_terms(d0, g4, A, B);
            const float4 col = lds4(a_col + 16 * slot);
#if BWD_PACK2
            float pw[4], ogv[4], dv[4];
            pair_alpha_bl2(fpy[0], fpy[1], g4.y, A, B, h4, pw[0], pw[1], ogv[0], ogv[1], dv[0], dv[1]);
            pair_alpha_bl2(fpy[2], fpy[3], g4.y, A, B, h4, pw[2], pw[3], ogv[2], ogv[3], dv[2], dv[3]);
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const float a = fminf(ogv[q], 0.99f);
                if (jj < last[q] && !(pw[q] > 0.0f) && a >= (1.0f / 255.0f)) {
                    const float wc = fmaf(wb[q], col.z, fmaf(wg[q], col.y, wr[q] * col.x));
                    pair_grad(a, ogv[q], dv[q], wc, wr[q], wg[q], wb[q], T[q], Q[q], v, s0, s1, s2);
                }
            }
#else
#pragma unroll
            for (int q = 0; q < 4; q++) {
#if BWD_FLAT_ALPHA
                // the exponent for every pixel (no early-exit branch), one
                // branch per pixel on the forward's exact decision
                const float d1 = fpy[q] - g4.y;
                const float power = __fmaf_rn(d1, __fmaf_rn(h4.x, d1, B), A);
                const float og = __fmul_rn(h4.z, ex2a(power));
                const float a = fminf(og, 0.99f);
                if (jj < last[q] && !(power > 0.0f) && a >= (1.0f / 255.0f)) {
                    const float wc = fmaf(wb[q], col.z, fmaf(wg[q], col.y, wr[q] * col.x));
                    pair_grad(a, og, d1, wc, wr[q], wg[q], wb[q], T[q], Q[q], v, s0, s1, s2);
                }
#else
                if (jj < last[q]) {
                    float og;
                    const float d1 = fpy[q] - g4.y;
                    const float a = pair_alpha(d1, A, B, h4, og);
                    if (a > 0.0f) {
                        const float wc = fmaf(wb[q], col.z, fmaf(wg[q], col.y, wr[q] * col.x));
                        pair_grad(a, og, d1, wc, wr[q], wg[q], wb[q], T[q], Q[q], v, s0, s1, s2);
                    }
                }
#endif
            }
#endif
            moment_terms(d0, s0, s1, s2, v);
            const float y = bfly9(v, lane);
            if (my_slot >= 0) sts(a_red + 36u * (uint32_t)slot, y);
        }
        // publish this warp's sums for the batch; the last warp to arrive folds
        if (lane == 0) spres[rs][warp] = bal;
        __threadfence_block();
        __syncwarp();
        int prev = 0;
        if (lane == 0) prev = atomicAdd(&sarrive[rs], 1);
        prev = __shfl_sync(FULL, prev, 0);
        if (prev == NH - 1) {
            __threadfence_block();
            const int jf = start + lane;
            if (jf < end) {
                const int32_t ent = entries[e0 + jf];
                const int rank = slot_rank ? slot_rank[ent] : ent;
                int64_t slot;
                if (slot_rank) {
                    slot = ent;  // live-only layout: the list entry is the slot
                } else if (emit_off) {
                    const int4 rc = rect_sorted[rank];
                    slot = emit_off[rank] + (int64_t)(ty - max(rc.y, row_lo)) * (rc.z - rc.x + 1) +
                           (tx - rc.x);
                } else {
                    slot = (int64_t)e0 + jf;
                }
                float4 *dst = reinterpret_cast<float4 *>(partials + PSTRIDE * slot);
                unsigned pm = 0u;
#pragma unroll
                for (int w = 0; w < NH; w++) pm |= ((spres[rs][w] >> lane) & 1u) << w;
                // live-only records carry their tile row (the fold's block key)
                const float rowf = slot_rank ? __int_as_float(ty) : 0.0f;
                if (pm == 0u) {
                    const float4 z = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                    dst[0] = z;
                    dst[1] = z;
                    dst[2] = make_float4(0.0f, rowf, 0.0f, 0.0f);
                } else {
                    float acc[9];
#pragma unroll
                    for (int q = 0; q < 9; q++) acc[q] = 0.0f;
#pragma unroll
                    for (int w = 0; w < NH; w++)
                        if ((pm >> w) & 1u) {
#pragma unroll
                            for (int q = 0; q < 9; q++) acc[q] += sred[rs][w][lane][q];
                        }
                    // the conic (a, b, c) and opacity of the entry, as preprocessed
                    const float4 f0 = __ldg(reinterpret_cast<const float4 *>(feat) + 3 * (int64_t)rank);
                    const float2 f1 = __ldg(reinterpret_cast<const float2 *>(feat + 12 * (int64_t)rank + 4));
                    const float ca = f0.z, cb = f0.w, cc = f1.x;
                    dst[0] = make_float4(fmaf(ca, acc[0], cb * acc[1]), fmaf(cb, acc[0], cc * acc[1]),
                                         -0.5f * acc[2], -acc[3]);
                    dst[1] = make_float4(-0.5f * acc[4], acc[5], acc[6], acc[7]);
                    // staged entries have o >= 1/255 (box_dead drops the rest)
                    dst[2] = make_float4(__fdiv_rn(acc[8], f1.y), rowf, 0.0f, 0.0f);
                }
            }
            __syncwarp();
            if (lane == 0) {
                sarrive[rs] = 0;
                __threadfence_block();
                *reinterpret_cast<volatile int *>(&sfolded[rs]) = bi;
            }
        }
        __syncwarp();  // the slice is restaged next batch
    }
}

}  // namespace f32

void launch_raster_fwd_f32(int n_tiles, int W, int H, int tiles_x, int row_lo,
                           const int32_t *tile_ids, const int32_t *tile_order,
                           const int32_t *offsets, const int32_t *entries,
                           const float *feat, float bg0, float bg1, float bg2, void *image,
                           int image_f64, float *t_final, int32_t *n_last, int32_t *n_contrib,
                           int32_t *n_iter, int64_t *touched, uint32_t *cmask,
                           const ChunkArgs *ch, const int32_t *slot_rank, cudaStream_t s) {
    const int mode = (touched ? f32::F_TOUCH : 0) | (n_contrib || n_iter ? f32::F_STATS : 0);
    const int chunk = ch ? ch->chunk : 0;
    float4 *cstate = ch && ch->chunk ? (float4 *)ch->state : nullptr;
    int32_t *qlast = ch && ch->chunk ? ch->tile_last : nullptr;
#define ISG_FWD(M)                                                                               \
    f32::fwd_kernel<M><<<n_tiles, f32::NT, 0, s>>>(W, H, tiles_x, row_lo, tile_ids, tile_order,  \
                                                   offsets,                                      \
                                                   entries, feat, bg0, bg1, bg2, image,          \
                                                   image_f64, t_final, n_last, n_contrib, n_iter, \
                                                   touched, cmask, chunk, cstate, qlast,       \
                                                   slot_rank)
    switch (mode) {
        case 0: ISG_FWD(0); break;
        case 1: ISG_FWD(1); break;
        case 2: ISG_FWD(2); break;
        default: ISG_FWD(3); break;
    }
#undef ISG_FWD
}

template <typename DL>
void launch_raster_bwd_f32(int n_tiles, int W, int H, int tiles_x, int row_lo,
                           const int32_t *tile_ids, const int32_t *tile_order,
                           const int32_t *offsets, const int32_t *entries,
                           const float *feat, const int4 *rect_sorted, const int64_t *emit_off,
                           float bg0, float bg1, float bg2, const float *t_final,
                           const int32_t *n_last, const DL *dl, float *partials,
                           const uint32_t *cmask, const ChunkArgs *ch, const int32_t *slot_rank,
                           cudaStream_t s) {
    const bool chunked = ch && ch->chunk;
    const int grid = chunked ? ch->max_items : n_tiles;
    const int2 *items = chunked ? (const int2 *)ch->items : nullptr;
    const int32_t *n_items = chunked ? ch->n_items : nullptr;
    const int chunk = chunked ? ch->chunk : 0;
    const float4 *cstate = chunked ? (const float4 *)ch->state : nullptr;
    const float *image = chunked ? ch->image : nullptr;
#define ISG_BWD32(MASK, CH, U)                                                               \
    f32::bwd_kernel<DL, MASK, CH, U><<<grid, f32::BNT, 0, s>>>(                                  \
        W, H, tiles_x, row_lo, tile_ids, tile_order, offsets, entries, feat, rect_sorted,        \
        emit_off, bg0, bg1, bg2, t_final, n_last, dl, partials, MASK ? cmask : nullptr, items,    \
        n_items, chunk, cstate, image, slot_rank)
    if (cmask) {
        if (chunked && ch->unroll2) ISG_BWD32(true, true, BWD_UNR);
        else if (chunked) ISG_BWD32(true, true, 1);
        else if (ch && ch->unroll2) ISG_BWD32(true, false, BWD_UNR);
        else ISG_BWD32(true, false, 1);
    } else {
        ISG_BWD32(false, false, 1);  // the unmasked launch is never chunked
    }
#undef ISG_BWD32
}

template void launch_raster_bwd_f32<float>(int, int, int, int, int, const int32_t *,
                                           const int32_t *,
                                           const int32_t *, const int32_t *, const float *,
                                           const int4 *, const int64_t *, float, float, float,
                                           const float *, const int32_t *, const float *, float *,
                                           const uint32_t *, const ChunkArgs *, const int32_t *,
                                           cudaStream_t);
template void launch_raster_bwd_f32<double>(int, int, int, int, int, const int32_t *,
                                            const int32_t *,
                                            const int32_t *, const int32_t *, const float *,
                                            const int4 *, const int64_t *, float, float, float,
                                            const float *, const int32_t *, const double *,
                                            float *, const uint32_t *, const ChunkArgs *,
                                            const int32_t *, cudaStream_t);

}  // namespace isg
