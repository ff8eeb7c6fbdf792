// project.cu -- per-Gaussian kernels on the float64 key path (sm_100a).
//
// Compiled with -fmad=false (see common.cuh): preprocess, chain rule, the
// fused chain+stats+Adam update and plain Adam.  All are one thread per
// Gaussian over SoA parameter rows; they are HBM-bound (92 B of parameters
// per Gaussian in, 48-96 B of raster features out; Adam streams 644 B per
// Gaussian) and the FP64 work per row (~250 flops for the projection,
// ~450 for the chain) stays well under the B200's FP64 rate.
#include <math.h>

#include "adam.cuh"
#include "common.cuh"

namespace isg {

template <typename F>
__device__ __forceinline__ void store_feat(F *base, const F (&v)[FEAT]);

template <>
__device__ __forceinline__ void store_feat<float>(float *base, const float (&v)[FEAT]) {
    float4 *b = reinterpret_cast<float4 *>(base);
    b[0] = make_float4(v[0], v[1], v[2], v[3]);
    b[1] = make_float4(v[4], v[5], v[6], v[7]);
    b[2] = make_float4(v[8], v[9], v[10], v[11]);
}

template <>
__device__ __forceinline__ void store_feat<double>(double *base, const double (&v)[FEAT]) {
    double2 *b = reinterpret_cast<double2 *>(base);
#pragma unroll
    for (int j = 0; j < 6; j++) b[j] = make_double2(v[2 * j], v[2 * j + 1]);
}

// _kernels.py:144-198 (+ the `keep` compaction flag of rasterizer.py:142-158).
template <typename P, typename F>
#ifndef PRE_MINB
#define PRE_MINB 8
#endif
__global__ void __launch_bounds__(128, PRE_MINB) preprocess_kernel(isg_params p, Cam cam_val, int tile,
                                                         int tiles_x, int tiles_y, uint64_t *key,
                                                         int4 *rect, F *feat, uint8_t *flag,
                                                         double *full64,
                                                         const Cam *__restrict__ cam_dev) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    // the camera by value, or from device memory (a graph-captured launch
    // whose camera is uploaded before each replay)
    const Cam cam = cam_dev ? *cam_dev : cam_val;
    Row<P> row;
    load_row<P>(p, i, row);
    Proj o;
    bool kept = false;
    int tx0 = 0, ty0 = 0, tx1 = -1, ty1 = -1;
    if (project_core<P>(row, p.degree, cam, o)) {
        const double u = o.u, v = o.v, r = o.radius;
        if (!(u + r < 0.0 || u - r > cam.width - 1.0 || v + r < 0.0 || v - r > cam.height - 1.0)) {
            // int(np.floor(x / tile)), clamped in double first so the int
            // conversion is always defined (same results after the clamps).
            double f0 = floor((u - r) / (double)tile), f1 = floor((u + r) / (double)tile);
            double g0 = floor((v - r) / (double)tile), g1 = floor((v + r) / (double)tile);
            f0 = fmin(fmax(f0, -1.0), (double)tiles_x);
            f1 = fmin(fmax(f1, -1.0), (double)tiles_x);
            g0 = fmin(fmax(g0, -1.0), (double)tiles_y);
            g1 = fmin(fmax(g1, -1.0), (double)tiles_y);
            tx0 = (int)f0; tx1 = (int)f1; ty0 = (int)g0; ty1 = (int)g1;
            if (!(tx1 < 0 || ty1 < 0 || tx0 >= tiles_x || ty0 >= tiles_y)) {
                kept = true;
                tx0 = max(tx0, 0);
                ty0 = max(ty0, 0);
                tx1 = min(tx1, tiles_x - 1);
                ty1 = min(ty1, tiles_y - 1);
            }
        }
    }
    flag[i] = kept ? 1 : 0;
    if (!kept) {
        key[i] = ~0ull;
        rect[i] = make_int4(0, 0, -1, -1);
    } else {
        key[i] = (uint64_t)__double_as_longlong(o.qz);
        rect[i] = make_int4(tx0, ty0, tx1, ty1);
        F v[FEAT] = {(F)o.u, (F)o.v, (F)o.ka, (F)o.kb, (F)o.kc, (F)o.opac,
                     (F)o.r, (F)o.g, (F)o.b, (F)0, (F)0, (F)0};
        store_feat<F>(feat + FEAT * i, v);
    }
    if (full64) {
        double *f = full64 + 16 * i;
        if (kept) {
            f[0] = o.u; f[1] = o.v; f[2] = o.ca; f[3] = o.cb; f[4] = o.cc;
            f[5] = o.ka; f[6] = o.kb; f[7] = o.kc; f[8] = o.qz;
            f[9] = o.r; f[10] = o.g; f[11] = o.b; f[12] = o.opac;
        } else {
            for (int j = 0; j < 13; j++) f[j] = 0.0;
        }
        f[13] = 0.0; f[14] = 0.0; f[15] = 0.0;
    }
}

// Parameter gradients of one Gaussian, in double (23 values:
// pos 3, log_scale 3, rot 4, logit 1, sh 12).  _kernels.py:415-634.
struct Grads {
    double pos[3], ls[3], rot[4], logit, sh[12];
};

__device__ __forceinline__ void zero_grads(Grads &out) {
#pragma unroll
    for (int j = 0; j < 3; j++) { out.pos[j] = 0.0; out.ls[j] = 0.0; }
#pragma unroll
    for (int j = 0; j < 4; j++) out.rot[j] = 0.0;
    out.logit = 0.0;
#pragma unroll
    for (int j = 0; j < 12; j++) out.sh[j] = 0.0;
}

template <typename P>
__device__ __forceinline__ bool chain_one(const Row<P> &row, int degree, const Cam &cam,
                                          const double *g2, Grads &out) {
    zero_grads(out);
    Proj o;
    if (!project_core<P>(row, degree, cam, o)) return false;
    const double *rot = cam.R;
    const double fx = cam.fx, fy = cam.fy;
    const double qcx = o.qx, qcy = o.qy, qcz = o.qz;
    const double con_a = o.ka, con_b = o.kb, con_c = o.kc, opac = o.opac;
    const double dirx = o.dx, diry = o.dy, dirz = o.dz, vlen = o.vlen;
    const double nqw = o.nw, nqx = o.nx, nqy = o.ny, nqz = o.nz, qnorm = o.qn;
    const double s20 = o.s0, s21 = o.s1, s22 = o.s2;
    const double r00 = o.r00, r01 = o.r01, r02 = o.r02, r10 = o.r10, r11 = o.r11, r12 = o.r12;
    const double r20 = o.r20, r21 = o.r21, r22 = o.r22;
    const double u00 = o.u00, u01 = o.u01, u02 = o.u02, u10 = o.u10, u11 = o.u11, u12 = o.u12;
    const double du = g2[0], dv = g2[1];
    const double dca = g2[2], dcb = g2[3], dcc = g2[4];
    double dcr = g2[5], dcg = g2[6], dcb_col = g2[7];
    const double dop = g2[8];
    const double *sh = row.sh;

    if (o.pr < 0.0 || o.pr > 1.0) dcr = 0.0;
    if (o.pg < 0.0 || o.pg > 1.0) dcg = 0.0;
    if (o.pb < 0.0 || o.pb > 1.0) dcb_col = 0.0;
    out.sh[0] = 0.0 + dcr * SH_C0;
    out.sh[1] = 0.0 + dcg * SH_C0;
    out.sh[2] = 0.0 + dcb_col * SH_C0;
    double ddirx = 0.0, ddiry = 0.0, ddirz = 0.0;
    if (degree >= 1) {
        out.sh[3] = 0.0 + dcr * (-SH_C1) * diry;
        out.sh[4] = 0.0 + dcg * (-SH_C1) * diry;
        out.sh[5] = 0.0 + dcb_col * (-SH_C1) * diry;
        out.sh[6] = 0.0 + dcr * SH_C1 * dirz;
        out.sh[7] = 0.0 + dcg * SH_C1 * dirz;
        out.sh[8] = 0.0 + dcb_col * SH_C1 * dirz;
        out.sh[9] = 0.0 + dcr * (-SH_C1) * dirx;
        out.sh[10] = 0.0 + dcg * (-SH_C1) * dirx;
        out.sh[11] = 0.0 + dcb_col * (-SH_C1) * dirx;
        ddirx = (-SH_C1) * (dcr * sh[9] + dcg * sh[10] + dcb_col * sh[11]);
        ddiry = (-SH_C1) * (dcr * sh[3] + dcg * sh[4] + dcb_col * sh[5]);
        ddirz = SH_C1 * (dcr * sh[6] + dcg * sh[7] + dcb_col * sh[8]);
    }
    double dot = dirx * ddirx + diry * ddiry + dirz * ddirz;
    double dpx = (ddirx - dirx * dot) / vlen;
    double dpy = (ddiry - diry * dot) / vlen;
    double dpz = (ddirz - dirz * dot) / vlen;

    out.logit = 0.0 + dop * opac * (1.0 - opac);

    double gh00 = dca, gh01 = 0.5 * dcb, gh11 = dcc;
    double t100 = con_a * gh00 + con_b * gh01;
    double t101 = con_a * gh01 + con_b * gh11;
    double t110 = con_b * gh00 + con_c * gh01;
    double t111 = con_b * gh01 + con_c * gh11;
    double k00 = -(t100 * con_a + t101 * con_b);
    double k01 = -(t100 * con_b + t101 * con_c);
    double k10 = -(t110 * con_a + t111 * con_b);
    double k11 = -(t110 * con_b + t111 * con_c);

    double gs00 = u00 * (k00 * u00 + k01 * u10) + u10 * (k10 * u00 + k11 * u10);
    double gs01 = u00 * (k00 * u01 + k01 * u11) + u10 * (k10 * u01 + k11 * u11);
    double gs02 = u00 * (k00 * u02 + k01 * u12) + u10 * (k10 * u02 + k11 * u12);
    double gs10 = u01 * (k00 * u00 + k01 * u10) + u11 * (k10 * u00 + k11 * u10);
    double gs11 = u01 * (k00 * u01 + k01 * u11) + u11 * (k10 * u01 + k11 * u11);
    double gs12 = u01 * (k00 * u02 + k01 * u12) + u11 * (k10 * u02 + k11 * u12);
    double gs20 = u02 * (k00 * u00 + k01 * u10) + u12 * (k10 * u00 + k11 * u10);
    double gs21 = u02 * (k00 * u01 + k01 * u11) + u12 * (k10 * u01 + k11 * u11);
    double gs22 = u02 * (k00 * u02 + k01 * u12) + u12 * (k10 * u02 + k11 * u12);

    double c3_00 = r00 * s20 * r00 + r01 * s21 * r01 + r02 * s22 * r02;
    double c3_01 = r00 * s20 * r10 + r01 * s21 * r11 + r02 * s22 * r12;
    double c3_02 = r00 * s20 * r20 + r01 * s21 * r21 + r02 * s22 * r22;
    double c3_11 = r10 * s20 * r10 + r11 * s21 * r11 + r12 * s22 * r12;
    double c3_12 = r10 * s20 * r20 + r11 * s21 * r21 + r12 * s22 * r22;
    double c3_22 = r20 * s20 * r20 + r21 * s21 * r21 + r22 * s22 * r22;
    double p00 = 2.0 * k00, p01 = k01 + k10, p11 = 2.0 * k11;
    double a00 = p00 * u00 + p01 * u10;
    double a01 = p00 * u01 + p01 * u11;
    double a02 = p00 * u02 + p01 * u12;
    double a10 = p01 * u00 + p11 * u10;
    double a11 = p01 * u01 + p11 * u11;
    double a12 = p01 * u02 + p11 * u12;
    double gu00 = a00 * c3_00 + a01 * c3_01 + a02 * c3_02;
    double gu01 = a00 * c3_01 + a01 * c3_11 + a02 * c3_12;
    double gu02 = a00 * c3_02 + a01 * c3_12 + a02 * c3_22;
    double gu10 = a10 * c3_00 + a11 * c3_01 + a12 * c3_02;
    double gu11 = a10 * c3_01 + a11 * c3_11 + a12 * c3_12;
    double gu12 = a10 * c3_02 + a11 * c3_12 + a12 * c3_22;

    double gj00 = gu00 * rot[0] + gu01 * rot[1] + gu02 * rot[2];
    double gj02 = gu00 * rot[6] + gu01 * rot[7] + gu02 * rot[8];
    double gj11 = gu10 * rot[3] + gu11 * rot[4] + gu12 * rot[5];
    double gj12 = gu10 * rot[6] + gu11 * rot[7] + gu12 * rot[8];

    double iz = 1.0 / qcz;
    double iz2 = iz * iz;
    double iz3 = iz2 * iz;
    double gq_x = du * (fx * iz) + gj02 * (-fx * iz2);
    double gq_y = dv * (fy * iz) + gj12 * (-fy * iz2);
    double gq_z = (du * (-fx * qcx * iz2) + dv * (-fy * qcy * iz2) + gj00 * (-fx * iz2) +
                   gj02 * (2.0 * fx * qcx * iz3) + gj11 * (-fy * iz2) +
                   gj12 * (2.0 * fy * qcy * iz3));
    dpx += rot[0] * gq_x + rot[3] * gq_y + rot[6] * gq_z;
    dpy += rot[1] * gq_x + rot[4] * gq_y + rot[7] * gq_z;
    dpz += rot[2] * gq_x + rot[5] * gq_y + rot[8] * gq_z;
    out.pos[0] = 0.0 + dpx;
    out.pos[1] = 0.0 + dpy;
    out.pos[2] = 0.0 + dpz;

    double dm0 = (r00 * (gs00 * r00 + gs01 * r10 + gs02 * r20) +
                  r10 * (gs10 * r00 + gs11 * r10 + gs12 * r20) +
                  r20 * (gs20 * r00 + gs21 * r10 + gs22 * r20));
    double dm1 = (r01 * (gs00 * r01 + gs01 * r11 + gs02 * r21) +
                  r11 * (gs10 * r01 + gs11 * r11 + gs12 * r21) +
                  r21 * (gs20 * r01 + gs21 * r11 + gs22 * r21));
    double dm2 = (r02 * (gs00 * r02 + gs01 * r12 + gs02 * r22) +
                  r12 * (gs10 * r02 + gs11 * r12 + gs12 * r22) +
                  r22 * (gs20 * r02 + gs21 * r12 + gs22 * r22));
    out.ls[0] = 0.0 + dm0 * 2.0 * s20;
    out.ls[1] = 0.0 + dm1 * 2.0 * s21;
    out.ls[2] = 0.0 + dm2 * 2.0 * s22;

    double q00 = gs00 + gs00, q01 = gs01 + gs10, q02 = gs02 + gs20;
    double q11 = gs11 + gs11, q12 = gs12 + gs21, q22 = gs22 + gs22;
    double gr00 = (q00 * r00 + q01 * r10 + q02 * r20) * s20;
    double gr01 = (q00 * r01 + q01 * r11 + q02 * r21) * s21;
    double gr02 = (q00 * r02 + q01 * r12 + q02 * r22) * s22;
    double gr10 = (q01 * r00 + q11 * r10 + q12 * r20) * s20;
    double gr11 = (q01 * r01 + q11 * r11 + q12 * r21) * s21;
    double gr12 = (q01 * r02 + q11 * r12 + q12 * r22) * s22;
    double gr20 = (q02 * r00 + q12 * r10 + q22 * r20) * s20;
    double gr21 = (q02 * r01 + q12 * r11 + q22 * r21) * s21;
    double gr22 = (q02 * r02 + q12 * r12 + q22 * r22) * s22;

    double dnw = 2.0 * (gr01 * (-nqz) + gr02 * nqy + gr10 * nqz + gr12 * (-nqx) +
                        gr20 * (-nqy) + gr21 * nqx);
    double dnx = 2.0 * (gr01 * nqy + gr02 * nqz + gr10 * nqy + gr11 * (-2.0 * nqx) +
                        gr12 * (-nqw) + gr20 * nqz + gr21 * nqw + gr22 * (-2.0 * nqx));
    double dny = 2.0 * (gr00 * (-2.0 * nqy) + gr01 * nqx + gr02 * nqw + gr10 * nqx +
                        gr12 * nqz + gr20 * (-nqw) + gr21 * nqz + gr22 * (-2.0 * nqy));
    double dnz = 2.0 * (gr00 * (-2.0 * nqz) + gr01 * (-nqw) + gr02 * nqx + gr10 * nqw +
                        gr11 * (-2.0 * nqz) + gr12 * nqy + gr20 * nqx + gr21 * nqy);
    double ndot = nqw * dnw + nqx * dnx + nqy * dny + nqz * dnz;
    out.rot[0] = 0.0 + (dnw - nqw * ndot) / qnorm;
    out.rot[1] = 0.0 + (dnx - nqx * ndot) / qnorm;
    out.rot[2] = 0.0 + (dny - nqy * ndot) / qnorm;
    out.rot[3] = 0.0 + (dnz - nqz * ndot) / qnorm;
    return true;
}

// rasterizer.py:248-280 (chain_to_params) with the final astype(dtype).
template <typename P>
__global__ void __launch_bounds__(256) chain_kernel(isg_params p, Cam cam, const uint8_t *flag,
                                                    const double *grad2d, P *dpos, P *dls,
                                                    P *drot, P *dlogit, P *dsh) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    Grads g;
    Row<P> row;
    if (flag[i]) {
        load_row<P>(p, i, row);
        chain_one<P>(row, p.degree, cam, grad2d + 9 * i, g);
    } else {
        zero_grads(g);
    }
    for (int j = 0; j < 3; j++) {
        dpos[3 * i + j] = (P)g.pos[j];
        dls[3 * i + j] = (P)g.ls[j];
    }
    for (int j = 0; j < 4; j++) drot[4 * i + j] = (P)g.rot[j];
    dlogit[i] = (P)g.logit;
    if (p.degree >= 1) {
#pragma unroll
        for (int j = 0; j < 12; j++) dsh[12 * i + j] = (P)g.sh[j];
    } else {
#pragma unroll
        for (int j = 0; j < 3; j++) dsh[3 * i + j] = (P)g.sh[j];
    }
}


// Fused: chain (flagged rows) + TrainStats (engine.py:508-515) + dense Adam
// over the five groups (engine.py:524-536, optim.py:20-56).  K3 = 3 (SH
// degree 0) or 12 (degree 1) keeps every index static (no local memory); the
// launch bound caps registers at 128 so 4 CTAs of 128 threads stay resident.
template <int K3>
__global__ void __launch_bounds__(128, 4) chain_adam_kernel(isg_train_state s, Cam cam,
                                                         const uint8_t *flag,
                                                         const double *grad2d, float lr0,
                                                         float lr1, float lr2, float lr3,
                                                         float lr4, AdamF c, double half_w,
                                                         double half_h) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= s.n) return;
    isg_params p;
    p.positions = s.positions;
    p.log_scales = s.log_scales;
    p.rotations = s.rotations;
    p.opacity_logits = s.opacity_logits;
    p.sh = s.sh;
    p.n = s.n;
    p.degree = s.degree;
    p.dtype = ISG_F32;
    Row<float> row;
    load_row<float>(p, i, row);
    Grads g;
    const bool vis = flag[i] != 0;
    if (vis) {
        const double *g2 = grad2d + 9 * i;
        chain_one<float>(row, s.degree, cam, g2, g);
        if (s.seen) s.seen[i] += 1;
        if (s.grad_accum) s.grad_accum[i] += hypot(g2[0] * half_w, g2[1] * half_h);
    } else {
        zero_grads(g);
    }
    // Parameters were read into `row` (as double) for the chain; Adam uses the
    // stored float32 values.
#pragma unroll
    for (int j = 0; j < 3; j++) {
        adam_f32(s.positions[3 * i + j], s.m_positions[3 * i + j], s.v_positions[3 * i + j],
                 (float)g.pos[j], lr0, c);
        adam_f32(s.log_scales[3 * i + j], s.m_log_scales[3 * i + j], s.v_log_scales[3 * i + j],
                 (float)g.ls[j], lr1, c);
    }
#pragma unroll
    for (int j = 0; j < 4; j++)
        adam_f32(s.rotations[4 * i + j], s.m_rotations[4 * i + j], s.v_rotations[4 * i + j],
                 (float)g.rot[j], lr2, c);
    adam_f32(s.opacity_logits[i], s.m_opacity_logits[i], s.v_opacity_logits[i],
             (float)g.logit, lr3, c);
#pragma unroll
    for (int j = 0; j < K3; j++) {
        const int64_t o = (int64_t)K3 * i + j;
        adam_f32(s.sh[o], s.m_sh[o], s.v_sh[o], (float)g.sh[j], lr4, c);
    }
}

// Chain rule + TrainStats for float32 parameters (training step, split from
// Adam so each kernel keeps its occupancy): grads written for every row
// (zeros for unflagged rows), stats for flagged rows.
template <int K3>
#ifndef CHAIN_MINB
#define CHAIN_MINB 4
#endif
__global__ void __launch_bounds__(128, CHAIN_MINB) chain_train_kernel(isg_params p, Cam cam,
                                                          const uint8_t *__restrict__ flag,
                                                          const int32_t *__restrict__ rank_of,
                                                          const double *__restrict__ grad2d,
                                                          float *dpos, float *dls, float *drot,
                                                          float *dlogit, float *dsh,
                                                          int64_t *seen, double *grad_accum,
                                                          double half_w, double half_h) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    Grads g;
    // rank_of: rank-ordered grad2d (row i -> its rank, -1 = not visible)
    const int64_t gi = rank_of ? (int64_t)rank_of[i] : (flag[i] ? i : -1);
    if (gi >= 0) {
        Row<float> row;
        load_row<float>(p, i, row);
        const double *g2 = grad2d + 9 * gi;
        chain_one<float>(row, p.degree, cam, g2, g);
        if (seen) seen[i] += 1;
        if (grad_accum) grad_accum[i] += hypot(g2[0] * half_w, g2[1] * half_h);
    } else {
        zero_grads(g);
    }
#pragma unroll
    for (int j = 0; j < 3; j++) {
        dpos[3 * i + j] = (float)g.pos[j];
        dls[3 * i + j] = (float)g.ls[j];
    }
#pragma unroll
    for (int j = 0; j < 4; j++) drot[4 * i + j] = (float)g.rot[j];
    dlogit[i] = (float)g.logit;
#pragma unroll
    for (int j = 0; j < K3; j++) dsh[(int64_t)K3 * i + j] = (float)g.sh[j];
}

// Dense Adam over up to 8 float32 groups in one launch, 4 elements per thread
// (16-byte vector accesses), numpy operation order (no FMA).
struct AdamGroups {
    float *p[8];
    const float *g[8];
    float *m[8];
    float *v[8];
    float lr[8];
    int64_t start[9];  // prefix of group sizes in float4 units
    int64_t n[8];      // group sizes in floats
    int count;
};

__global__ void __launch_bounds__(256) adam_groups_kernel(AdamGroups G, AdamF c) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= G.start[G.count]) return;
    int k = 0;
#pragma unroll
    for (int j = 1; j < 8; j++)
        if (j < G.count && q >= G.start[j]) k = j;
    const int64_t e = 4 * (q - G.start[k]);
    const int64_t n = G.n[k];
    const float lr = G.lr[k];
    if (e + 4 <= n && (((uintptr_t)G.p[k] | (uintptr_t)G.g[k] | (uintptr_t)G.m[k] |
                        (uintptr_t)G.v[k]) & 15) == 0) {
        float4 p = *reinterpret_cast<float4 *>(G.p[k] + e);
        const float4 g = *reinterpret_cast<const float4 *>(G.g[k] + e);
        float4 m = *reinterpret_cast<float4 *>(G.m[k] + e);
        float4 v = *reinterpret_cast<float4 *>(G.v[k] + e);
        adam_f32(p.x, m.x, v.x, g.x, lr, c);
        adam_f32(p.y, m.y, v.y, g.y, lr, c);
        adam_f32(p.z, m.z, v.z, g.z, lr, c);
        adam_f32(p.w, m.w, v.w, g.w, lr, c);
        *reinterpret_cast<float4 *>(G.p[k] + e) = p;
        *reinterpret_cast<float4 *>(G.m[k] + e) = m;
        *reinterpret_cast<float4 *>(G.v[k] + e) = v;
    } else {
        for (int64_t j = e; j < e + 4 && j < n; j++)
            adam_f32(G.p[k][j], G.m[k][j], G.v[k][j], G.g[k][j], lr, c);
    }
}

template <typename T>
__global__ void __launch_bounds__(256) adam_kernel(int64_t n, T *p, const T *g, T *m, T *v, T b1,
                                                   T omb1, T b2, T omb2, T bc1, T bc2, T lr,
                                                   T eps) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    T gi = g[i];
    T mi = m[i] * b1;
    mi = mi + omb1 * gi;
    T vi = v[i] * b2;
    T gg = gi * gi;
    vi = vi + omb2 * gg;
    T mhat = mi / bc1;
    T vhat = vi / bc2;
    T den = sqrt(vhat) + eps;
    T step = (lr * mhat) / den;
    p[i] = p[i] - step;
    m[i] = mi;
    v[i] = vi;
}

__global__ void exp_kernel(int64_t n, const double *x, double *y) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = exp_glibc(x[i]);
}

// densify_and_prune's classification (training.py:334-347), statement for
// statement in float64 with the glibc-exact exp (the reference's numpy):
//   avg = grad_accum / max(seen, 1); scales = exp(log_scales); opacity =
//   1 / (1 + exp(-logit)); prune = opacity < opacity_prune (| max scale >
//   scale_prune when finite); hot = avg > grad_thr & !prune; split = hot &
//   max scale > split_thr; clone = hot & !split.  cls: 0 keep, 1 clone,
//   2 split, 3 prune.
__global__ void densify_classify_kernel(int64_t n, const float *__restrict__ log_scales,
                                        const float *__restrict__ logits,
                                        const int64_t *__restrict__ seen,
                                        const double *__restrict__ grad_accum,
                                        double opacity_prune, double scale_prune,
                                        int scale_prune_on, double grad_thr, double split_thr,
                                        uint8_t *__restrict__ cls) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t s = seen[i];
    const double avg = grad_accum[i] / (double)(s > 1 ? s : 1);
    double mx = exp_glibc((double)log_scales[3 * i]);
    mx = fmax(mx, exp_glibc((double)log_scales[3 * i + 1]));
    mx = fmax(mx, exp_glibc((double)log_scales[3 * i + 2]));
    const double opacity = 1.0 / (1.0 + exp_glibc(-(double)logits[i]));
    bool prune = opacity < opacity_prune;
    if (scale_prune_on) prune = prune || mx > scale_prune;
    const bool hot = avg > grad_thr && !prune;
    const bool split = hot && mx > split_thr;
    cls[i] = prune ? 3 : split ? 2 : hot ? 1 : 0;
}

}  // namespace isg

using namespace isg;

extern "C" int isg_preprocess(const isg_params *p, const isg_camera *cam, int32_t tile_size,
                              const isg_preprocess_out *out, void *stream) {
    if (!p || !cam || !out || tile_size != TILE || p->n < 0) return (int)cudaErrorInvalidValue;
    if (p->n == 0) return 0;
    if (!out->key || !out->rect || !out->flag || !out->feat) return (int)cudaErrorInvalidValue;
    Cam c = to_cam(*cam);
    int tiles_x = (cam->width + tile_size - 1) / tile_size;
    int tiles_y = (cam->height + tile_size - 1) / tile_size;
    cudaStream_t s = (cudaStream_t)stream;
    dim3 grid(blocks_for(p->n, 128));
    int4 *rect = reinterpret_cast<int4 *>(out->rect);
    if (p->dtype == ISG_F32 && out->feat_dtype == ISG_F32)
        preprocess_kernel<float, float><<<grid, 128, 0, s>>>(*p, c, tile_size, tiles_x, tiles_y,
                                                             out->key, rect, (float *)out->feat,
                                                             out->flag, out->full64, nullptr);
    else if (p->dtype == ISG_F32 && out->feat_dtype == ISG_F64)
        preprocess_kernel<float, double><<<grid, 128, 0, s>>>(*p, c, tile_size, tiles_x, tiles_y,
                                                              out->key, rect, (double *)out->feat,
                                                              out->flag, out->full64, nullptr);
    else if (p->dtype == ISG_F64 && out->feat_dtype == ISG_F32)
        preprocess_kernel<double, float><<<grid, 128, 0, s>>>(*p, c, tile_size, tiles_x, tiles_y,
                                                              out->key, rect, (float *)out->feat,
                                                              out->flag, out->full64, nullptr);
    else if (p->dtype == ISG_F64 && out->feat_dtype == ISG_F64)
        preprocess_kernel<double, double><<<grid, 128, 0, s>>>(
            *p, c, tile_size, tiles_x, tiles_y, out->key, rect, (double *)out->feat, out->flag,
            out->full64, nullptr);
    else
        return (int)cudaErrorInvalidValue;
    ISG_CHECK_LAUNCH();
    return 0;
}

// isg_preprocess with the camera read from device memory (an isg_camera
// there, uploaded by the caller before the launch): the launch can be
// captured into a CUDA graph and replayed for any view.  Float32 parameters
// and features.
extern "C" int isg_preprocess_devcam(const isg_params *p, const isg_camera *cam_dev,
                                     int32_t width, int32_t height, int32_t tile_size,
                                     const isg_preprocess_out *out, void *stream) {
    static_assert(sizeof(Cam) == sizeof(isg_camera), "Cam mirrors isg_camera");
    if (!p || !cam_dev || !out || tile_size != TILE || p->n < 0 || width <= 0 || height <= 0 ||
        p->dtype != ISG_F32 || out->feat_dtype != ISG_F32)
        return (int)cudaErrorInvalidValue;
    if (p->n == 0) return 0;
    if (!out->key || !out->rect || !out->flag || !out->feat) return (int)cudaErrorInvalidValue;
    const int tiles_x = (width + tile_size - 1) / tile_size;
    const int tiles_y = (height + tile_size - 1) / tile_size;
    preprocess_kernel<float, float><<<dim3(blocks_for(p->n, 128)), 128, 0, (cudaStream_t)stream>>>(
        *p, Cam{}, tile_size, tiles_x, tiles_y, out->key, reinterpret_cast<int4 *>(out->rect),
        (float *)out->feat, out->flag, out->full64, reinterpret_cast<const Cam *>(cam_dev));
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_chain(const isg_params *p, const isg_camera *cam, const uint8_t *flag,
                         const double *grad2d, void *d_positions, void *d_log_scales,
                         void *d_rotations, void *d_opacity_logits, void *d_sh, void *stream) {
    if (!p || !cam || p->n < 0) return (int)cudaErrorInvalidValue;
    if (p->n == 0) return 0;
    Cam c = to_cam(*cam);
    cudaStream_t s = (cudaStream_t)stream;
    dim3 grid(blocks_for(p->n, 256));
    if (p->dtype == ISG_F32)
        chain_kernel<float><<<grid, 256, 0, s>>>(*p, c, flag, grad2d, (float *)d_positions,
                                                 (float *)d_log_scales, (float *)d_rotations,
                                                 (float *)d_opacity_logits, (float *)d_sh);
    else if (p->dtype == ISG_F64)
        chain_kernel<double><<<grid, 256, 0, s>>>(*p, c, flag, grad2d, (double *)d_positions,
                                                  (double *)d_log_scales, (double *)d_rotations,
                                                  (double *)d_opacity_logits, (double *)d_sh);
    else
        return (int)cudaErrorInvalidValue;
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_adam(int32_t dtype, int64_t n, void *p, const void *g, void *m, void *v,
                        const isg_adam_consts *c, void *stream) {
    if (!c || n < 0) return (int)cudaErrorInvalidValue;
    if (n == 0) return 0;
    cudaStream_t s = (cudaStream_t)stream;
    dim3 grid(blocks_for(n, 256));
    if (dtype == ISG_F32)
        adam_kernel<float><<<grid, 256, 0, s>>>(n, (float *)p, (const float *)g, (float *)m,
                                                (float *)v, (float)c->b1, (float)c->omb1,
                                                (float)c->b2, (float)c->omb2, (float)c->bc1,
                                                (float)c->bc2, (float)c->lr, (float)c->eps);
    else if (dtype == ISG_F64)
        adam_kernel<double><<<grid, 256, 0, s>>>(n, (double *)p, (const double *)g, (double *)m,
                                                 (double *)v, c->b1, c->omb1, c->b2, c->omb2,
                                                 c->bc1, c->bc2, c->lr, c->eps);
    else
        return (int)cudaErrorInvalidValue;
    ISG_CHECK_LAUNCH();
    return 0;
}

static int chain_train_launch(const isg_params *p, const isg_camera *cam, const uint8_t *flag,
                              const int32_t *rank_of, const double *grad2d, float *d_positions,
                              float *d_log_scales, float *d_rotations, float *d_opacity_logits,
                              float *d_sh, int64_t *seen, double *grad_accum, double half_w,
                              double half_h, void *stream);
namespace isg {
void launch_chain_train_f32(const isg_params &p, const Cam &cam, const uint8_t *flag,
                            const int32_t *rank_of, const double *grad2d, float *dpos,
                            float *dls, float *drot, float *dlogit, float *dsh, int64_t *seen,
                            double *grad_accum, double half_w, double half_h, cudaStream_t s);
}

extern "C" int isg_chain_train(const isg_params *p, const isg_camera *cam, const uint8_t *flag,
                               const double *grad2d, float *d_positions, float *d_log_scales,
                               float *d_rotations, float *d_opacity_logits, float *d_sh,
                               int64_t *seen, double *grad_accum, double half_w, double half_h,
                               void *stream) {
    if (!flag) return (int)cudaErrorInvalidValue;
    return chain_train_launch(p, cam, flag, nullptr, grad2d, d_positions, d_log_scales,
                              d_rotations, d_opacity_logits, d_sh, seen, grad_accum, half_w,
                              half_h, stream);
}

namespace isg {
void launch_chain_fold_train_f32(const isg_params &p, const Cam &cam, const int32_t *rank_of,
                                 const int64_t *live_off, const float *partials,
                                 const int32_t *rect_sorted, int row_lo, int row_hi, int canon,
                                 double *grad2d_out, float *dpos, float *dls, float *drot,
                                 float *dlogit, float *dsh, int64_t *seen, double *grad_accum,
                                 double half_w, double half_h, cudaStream_t s);
}

namespace isg {
void launch_chain_fold_adam_f32(const isg_train_state &st, const Cam &cam, const uint8_t *flag,
                                const double *grad2d, const int32_t *rank_of,
                                const int64_t *live_off, const float *partials,
                                const int32_t *rect_sorted, int row_lo, int row_hi, int canon,
                                double *grad2d_out, float *const *grads_out, const float *lr5,
                                const isg_adam_consts &ac, double half_w, double half_h,
                                cudaStream_t s);
}

// The fused Adam updates each CTA's rows with 16-byte accesses.
static bool state_aligned16(const isg_train_state &s) {
    const void *ptrs[15] = {s.positions,   s.log_scales,       s.rotations,     s.opacity_logits,
                            s.sh,          s.m_positions,      s.m_log_scales,  s.m_rotations,
                            s.m_opacity_logits, s.m_sh,        s.v_positions,   s.v_log_scales,
                            s.v_rotations, s.v_opacity_logits, s.v_sh};
    for (const void *q : ptrs)
        if (!q || (reinterpret_cast<uintptr_t>(q) & 15) != 0) return false;
    return true;
}

extern "C" int isg_chain_fold_adam(const isg_train_state *st, const isg_camera *cam,
                                   const int32_t *rank_of, const int64_t *live_off,
                                   const float *partials, const int32_t *rect_sorted,
                                   int32_t row_lo, int32_t row_hi, int32_t canon_rows,
                                   double *grad2d_out, float *const *grads_out, const float *lr5,
                                   const isg_adam_consts *c, double half_w, double half_h,
                                   void *stream) {
    if (!st || !cam || !rank_of || !live_off || !partials || !rect_sorted || canon_rows < 1 ||
        st->n < 0 || !lr5 || !c)
        return (int)cudaErrorInvalidValue;
    if (grads_out)
        for (int k = 0; k < 5; k++)
            if (!grads_out[k]) return (int)cudaErrorInvalidValue;
    if (!state_aligned16(*st)) return (int)cudaErrorInvalidValue;
    if (st->n == 0) return 0;
    launch_chain_fold_adam_f32(*st, to_cam(*cam), nullptr, nullptr, rank_of, live_off, partials,
                               rect_sorted, row_lo, row_hi, canon_rows, grad2d_out, grads_out, lr5,
                               *c, half_w, half_h, (cudaStream_t)stream);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_chain_adam_train(const isg_train_state *st, const isg_camera *cam,
                                    const uint8_t *flag, const double *grad2d,
                                    float *const *grads_out, const float *lr5,
                                    const isg_adam_consts *c, double half_w, double half_h,
                                    void *stream) {
    if (!st || !cam || !flag || !grad2d || st->n < 0 || !lr5 || !c)
        return (int)cudaErrorInvalidValue;
    if (grads_out)
        for (int k = 0; k < 5; k++)
            if (!grads_out[k]) return (int)cudaErrorInvalidValue;
    if (!state_aligned16(*st)) return (int)cudaErrorInvalidValue;
    if (st->n == 0) return 0;
    launch_chain_fold_adam_f32(*st, to_cam(*cam), flag, grad2d, nullptr, nullptr, nullptr, nullptr,
                               0, 0, 1, nullptr, grads_out, lr5, *c, half_w, half_h,
                               (cudaStream_t)stream);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_chain_fold_train(const isg_params *p, const isg_camera *cam,
                                    const int32_t *rank_of, const int64_t *live_off,
                                    const float *partials, const int32_t *rect_sorted,
                                    int32_t row_lo, int32_t row_hi, int32_t canon_rows,
                                    double *grad2d_out, float *d_positions, float *d_log_scales,
                                    float *d_rotations, float *d_opacity_logits, float *d_sh,
                                    int64_t *seen, double *grad_accum, double half_w,
                                    double half_h, void *stream) {
    if (!p || !cam || !rank_of || !live_off || !partials || !rect_sorted || canon_rows < 1 ||
        p->n < 0 || p->dtype != ISG_F32 || !d_positions || !d_log_scales || !d_rotations ||
        !d_opacity_logits || !d_sh)
        return (int)cudaErrorInvalidValue;
    if (p->n == 0) return 0;
    const Cam c = to_cam(*cam);
    launch_chain_fold_train_f32(*p, c, rank_of, live_off, partials, rect_sorted, row_lo, row_hi,
                                canon_rows, grad2d_out, d_positions, d_log_scales, d_rotations,
                                d_opacity_logits, d_sh, seen, grad_accum, half_w, half_h,
                                (cudaStream_t)stream);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_chain_train_ranked(const isg_params *p, const isg_camera *cam,
                                      const int32_t *rank_of, const double *grad2d_ranked,
                                      float *d_positions, float *d_log_scales,
                                      float *d_rotations, float *d_opacity_logits, float *d_sh,
                                      int64_t *seen, double *grad_accum, double half_w,
                                      double half_h, void *stream) {
    if (!rank_of) return (int)cudaErrorInvalidValue;
    return chain_train_launch(p, cam, nullptr, rank_of, grad2d_ranked, d_positions,
                              d_log_scales, d_rotations, d_opacity_logits, d_sh, seen, grad_accum,
                              half_w, half_h, stream);
}

static int chain_train_launch(const isg_params *p, const isg_camera *cam, const uint8_t *flag,
                              const int32_t *rank_of, const double *grad2d, float *d_positions,
                              float *d_log_scales, float *d_rotations, float *d_opacity_logits,
                              float *d_sh, int64_t *seen, double *grad_accum, double half_w,
                              double half_h, void *stream) {
    if (!p || !cam || !grad2d || p->n < 0 || p->dtype != ISG_F32)
        return (int)cudaErrorInvalidValue;
    if (p->n == 0) return 0;
    Cam c = to_cam(*cam);
    cudaStream_t s = (cudaStream_t)stream;
    // float32 chain (chain_f32.cu): the training step's gradients are float32
    launch_chain_train_f32(*p, c, flag, rank_of, grad2d, d_positions, d_log_scales, d_rotations,
                           d_opacity_logits, d_sh, seen, grad_accum, half_w, half_h, s);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_adam_groups(int32_t count, float *const *p, const float *const *g,
                               float *const *m, float *const *v, const int64_t *n,
                               const float *lr, const isg_adam_consts *c, void *stream) {
    if (count < 1 || count > 8 || !c) return (int)cudaErrorInvalidValue;
    AdamGroups G;
    G.count = count;
    G.start[0] = 0;
    for (int k = 0; k < count; k++) {
        G.p[k] = p[k];
        G.g[k] = g[k];
        G.m[k] = m[k];
        G.v[k] = v[k];
        G.lr[k] = lr[k];
        G.n[k] = n[k];
        G.start[k + 1] = G.start[k] + (n[k] + 3) / 4;
    }
    for (int k = count; k < 8; k++) {
        G.p[k] = nullptr;
        G.g[k] = nullptr;
        G.m[k] = G.v[k] = nullptr;
        G.lr[k] = 0.0f;
        G.n[k] = 0;
        G.start[k + 1] = G.start[count];
    }
    if (G.start[count] == 0) return 0;
    AdamF a{(float)c->b1, (float)c->omb1, (float)c->b2, (float)c->omb2,
            (float)c->bc1, (float)c->bc2, (float)c->eps};
    adam_groups_kernel<<<blocks_for(G.start[count], 256), 256, 0, (cudaStream_t)stream>>>(G, a);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_chain_adam(const isg_train_state *st, const isg_camera *cam,
                              const uint8_t *flag, const double *grad2d, const float *lr5,
                              const isg_adam_consts *c, double half_w, double half_h,
                              void *stream) {
    if (!st || !cam || !flag || !grad2d || !lr5 || !c || st->n < 0)
        return (int)cudaErrorInvalidValue;
    if (st->n == 0) return 0;
    Cam k = to_cam(*cam);
    AdamF a{(float)c->b1, (float)c->omb1, (float)c->b2, (float)c->omb2,
            (float)c->bc1, (float)c->bc2, (float)c->eps};
    cudaStream_t s = (cudaStream_t)stream;
    if (st->degree >= 1)
        chain_adam_kernel<12><<<blocks_for(st->n, 128), 128, 0, s>>>(
            *st, k, flag, grad2d, lr5[0], lr5[1], lr5[2], lr5[3], lr5[4], a, half_w, half_h);
    else
        chain_adam_kernel<3><<<blocks_for(st->n, 128), 128, 0, s>>>(
            *st, k, flag, grad2d, lr5[0], lr5[1], lr5[2], lr5[3], lr5[4], a, half_w, half_h);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_densify_classify(int64_t n, const float *log_scales, const float *logits,
                                    const int64_t *seen, const double *grad_accum,
                                    double opacity_prune, double scale_prune,
                                    int32_t scale_prune_on, double grad_threshold,
                                    double split_threshold, uint8_t *cls, void *stream) {
    if (n < 0 || (n > 0 && (!log_scales || !logits || !seen || !grad_accum || !cls)))
        return (int)cudaErrorInvalidValue;
    if (n == 0) return 0;
    densify_classify_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
        n, log_scales, logits, seen, grad_accum, opacity_prune, scale_prune, scale_prune_on,
        grad_threshold, split_threshold, cls);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_exp_f64(int64_t n, const double *x, double *y, void *stream) {
    if (n < 0) return (int)cudaErrorInvalidValue;
    if (n == 0) return 0;
    exp_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(n, x, y);
    ISG_CHECK_LAUNCH();
    return 0;
}
