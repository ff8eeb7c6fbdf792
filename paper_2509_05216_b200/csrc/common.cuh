// common.cuh -- shared device code for libisogs (B200, sm_100a).
//
// Constants and the float64 projection core shared by preprocess and the
// chain rule, so both see bit-identical intermediates exactly as the
// reference's _project_core is shared by _project_kernel and _chain_kernel
// (/root/reference/pkg/src/isosplat/_kernels.py:26-140, 144-198, 415-634).
// Translation units that include the projection core are compiled with
// -fmad=false: numba never contracts a*b+c into an FMA, and neither may we.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/isogs.h"
#include "glibc_exp.cuh"

namespace isg {

// _kernels.py:15-22
constexpr double SH_C0 = 0.28209479177387814;
constexpr double SH_C1 = 0.4886025119029199;
constexpr double NEAR_PLANE = 0.01;
constexpr double COV_DILATION = 0.3;
constexpr double ALPHA_CLAMP = 0.99;
constexpr double T_STOP = 1e-4;
constexpr int TILE = 16;
constexpr int FEAT = 12;  // raster features per splat (see isg_preprocess_out)

// Floats / doubles per (tile, splat) gradient subtotal record: 9 values
// (dmean 2, dconic 3, dcolor 3, dopac 1); float32 records are padded to 12
// (48 B, three 16-byte stores, 16-byte aligned), float64 records are packed.
template <typename T> constexpr int partial_stride();
template <> constexpr int partial_stride<float>() { return 12; }
template <> constexpr int partial_stride<double>() { return 9; }

struct Cam {
    double R[9];
    double t[3];
    double C[3];
    double fx, fy, cx, cy;
    int width, height;
};

inline Cam to_cam(const isg_camera &c) {
    Cam k;
    for (int i = 0; i < 9; i++) k.R[i] = c.R[i];
    for (int i = 0; i < 3; i++) {
        k.t[i] = c.t[i];
        k.C[i] = c.C[i];
    }
    k.fx = c.fx;
    k.fy = c.fy;
    k.cx = c.cx;
    k.cy = c.cy;
    k.width = c.width;
    k.height = c.height;
    return k;
}

// Every intermediate the chain rule needs (_kernels.py:29-35 tuple layout).
struct Proj {
    double qx, qy, qz, u, v;
    double ca, cb, cc, det;
    double ka, kb, kc, radius, opac;
    double r, g, b, pr, pg, pb;
    double dx, dy, dz, vlen;
    double nw, nx, ny, nz, qn;
    double s0, s1, s2;
    double r00, r01, r02, r10, r11, r12, r20, r21, r22;
    double u00, u01, u02, u10, u11, u12;
};

template <typename P>
struct Row {
    double px, py, pz, lsx, lsy, lsz, qw, qx, qy, qz, logit;
    double sh[12];
};

template <typename P>
__device__ __forceinline__ void load_row(const isg_params &p, int64_t i, Row<P> &r) {
    const P *pos = (const P *)p.positions;
    const P *ls = (const P *)p.log_scales;
    const P *rot = (const P *)p.rotations;
    const P *lg = (const P *)p.opacity_logits;
    const P *sh = (const P *)p.sh;
    r.px = (double)pos[3 * i];
    r.py = (double)pos[3 * i + 1];
    r.pz = (double)pos[3 * i + 2];
    r.lsx = (double)ls[3 * i];
    r.lsy = (double)ls[3 * i + 1];
    r.lsz = (double)ls[3 * i + 2];
    r.qw = (double)rot[4 * i];
    r.qx = (double)rot[4 * i + 1];
    r.qy = (double)rot[4 * i + 2];
    r.qz = (double)rot[4 * i + 3];
    r.logit = (double)lg[i];
    const int k3 = p.degree >= 1 ? 12 : 3;
#pragma unroll
    for (int j = 0; j < 12; j++) r.sh[j] = j < k3 ? (double)sh[(int64_t)k3 * i + j] : 0.0;
}

// _kernels.py:26-140, statement by statement, strict left-to-right float64.
// Compiled without FMA contraction (see file comment); exp is the glibc port.
template <typename P>
__device__ __forceinline__ bool project_core(const Row<P> &in, int degree, const Cam &cam,
                                             Proj &o) {
    const double *rot = cam.R;
    const double px = in.px, py = in.py, pz = in.pz;
    double qcx = rot[0] * px + rot[1] * py + rot[2] * pz + cam.t[0];
    double qcy = rot[3] * px + rot[4] * py + rot[5] * pz + cam.t[1];
    double qcz = rot[6] * px + rot[7] * py + rot[8] * pz + cam.t[2];
    if (qcz <= NEAR_PLANE) return false;
    const double qw = in.qw, qx = in.qx, qy = in.qy, qz = in.qz;
    double qnorm = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
    if (qnorm < 1e-12) return false;
    double nqw = qw / qnorm, nqx = qx / qnorm, nqy = qy / qnorm, nqz = qz / qnorm;
    double r00 = 1.0 - 2.0 * (nqy * nqy + nqz * nqz);
    double r01 = 2.0 * (nqx * nqy - nqw * nqz);
    double r02 = 2.0 * (nqx * nqz + nqw * nqy);
    double r10 = 2.0 * (nqx * nqy + nqw * nqz);
    double r11 = 1.0 - 2.0 * (nqx * nqx + nqz * nqz);
    double r12 = 2.0 * (nqy * nqz - nqw * nqx);
    double r20 = 2.0 * (nqx * nqz - nqw * nqy);
    double r21 = 2.0 * (nqy * nqz + nqw * nqx);
    double r22 = 1.0 - 2.0 * (nqx * nqx + nqy * nqy);
    double s20 = exp_glibc(2.0 * in.lsx);
    double s21 = exp_glibc(2.0 * in.lsy);
    double s22 = exp_glibc(2.0 * in.lsz);
    double c00 = r00 * s20 * r00 + r01 * s21 * r01 + r02 * s22 * r02;
    double c01 = r00 * s20 * r10 + r01 * s21 * r11 + r02 * s22 * r12;
    double c02 = r00 * s20 * r20 + r01 * s21 * r21 + r02 * s22 * r22;
    double c11 = r10 * s20 * r10 + r11 * s21 * r11 + r12 * s22 * r12;
    double c12 = r10 * s20 * r20 + r11 * s21 * r21 + r12 * s22 * r22;
    double c22 = r20 * s20 * r20 + r21 * s21 * r21 + r22 * s22 * r22;
    double iz = 1.0 / qcz;
    double iz2 = iz * iz;
    double j00 = cam.fx * iz;
    double j02 = -cam.fx * qcx * iz2;
    double j11 = cam.fy * iz;
    double j12 = -cam.fy * qcy * iz2;
    double u00 = j00 * rot[0] + j02 * rot[6];
    double u01 = j00 * rot[1] + j02 * rot[7];
    double u02 = j00 * rot[2] + j02 * rot[8];
    double u10 = j11 * rot[3] + j12 * rot[6];
    double u11 = j11 * rot[4] + j12 * rot[7];
    double u12 = j11 * rot[5] + j12 * rot[8];
    double w00 = u00 * c00 + u01 * c01 + u02 * c02;
    double w01 = u00 * c01 + u01 * c11 + u02 * c12;
    double w02 = u00 * c02 + u01 * c12 + u02 * c22;
    double w10 = u10 * c00 + u11 * c01 + u12 * c02;
    double w11 = u10 * c01 + u11 * c11 + u12 * c12;
    double w12 = u10 * c02 + u11 * c12 + u12 * c22;
    double ca = w00 * u00 + w01 * u01 + w02 * u02 + COV_DILATION;
    double cb = w00 * u10 + w01 * u11 + w02 * u12;
    double cc = w10 * u10 + w11 * u11 + w12 * u12 + COV_DILATION;
    double det = ca * cc - cb * cb;
    if (det <= 0.0) return false;
    double mid = 0.5 * (ca + cc);
    double disc = mid * mid - det;
    if (disc < 0.0) disc = 0.0;
    double lam = mid + sqrt(disc);
    o.radius = 3.0 * sqrt(lam);
    o.ka = cc / det;
    o.kb = -cb / det;
    o.kc = ca / det;
    o.u = cam.fx * qcx * iz + cam.cx;
    o.v = cam.fy * qcy * iz + cam.cy;
    o.opac = 1.0 / (1.0 + exp_glibc(-in.logit));
    double vx = px - cam.C[0], vy = py - cam.C[1], vz = pz - cam.C[2];
    double vlen = sqrt(vx * vx + vy * vy + vz * vz);
    if (vlen < 1e-12) return false;
    double dx = vx / vlen, dy = vy / vlen, dz = vz / vlen;
    const double *sh = in.sh;
    double pr = 0.5 + SH_C0 * sh[0];
    double pg = 0.5 + SH_C0 * sh[1];
    double pb = 0.5 + SH_C0 * sh[2];
    if (degree >= 1) {
        pr = pr + (-SH_C1) * dy * sh[3];
        pg = pg + (-SH_C1) * dy * sh[4];
        pb = pb + (-SH_C1) * dy * sh[5];
        pr = pr + SH_C1 * dz * sh[6];
        pg = pg + SH_C1 * dz * sh[7];
        pb = pb + SH_C1 * dz * sh[8];
        pr = pr + (-SH_C1) * dx * sh[9];
        pg = pg + (-SH_C1) * dx * sh[10];
        pb = pb + (-SH_C1) * dx * sh[11];
    }
    double cr = pr, cg = pg, cbl = pb;  // min(max(x, 0), 1), builtin semantics
    if (0.0 > cr) cr = 0.0;
    if (1.0 < cr) cr = 1.0;
    if (0.0 > cg) cg = 0.0;
    if (1.0 < cg) cg = 1.0;
    if (0.0 > cbl) cbl = 0.0;
    if (1.0 < cbl) cbl = 1.0;
    o.qx = qcx; o.qy = qcy; o.qz = qcz;
    o.ca = ca; o.cb = cb; o.cc = cc; o.det = det;
    o.r = cr; o.g = cg; o.b = cbl;
    o.pr = pr; o.pg = pg; o.pb = pb;
    o.dx = dx; o.dy = dy; o.dz = dz; o.vlen = vlen;
    o.nw = nqw; o.nx = nqx; o.ny = nqy; o.nz = nqz; o.qn = qnorm;
    o.s0 = s20; o.s1 = s21; o.s2 = s22;
    o.r00 = r00; o.r01 = r01; o.r02 = r02;
    o.r10 = r10; o.r11 = r11; o.r12 = r12;
    o.r20 = r20; o.r21 = r21; o.r22 = r22;
    o.u00 = u00; o.u01 = u01; o.u02 = u02;
    o.u10 = u10; o.u11 = u11; o.u12 = u12;
    return true;
}

inline int blocks_for(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    return (int)(b < 1 ? 1 : b);
}

}  // namespace isg

#define ISG_CHECK_LAUNCH() \
    do {                                    \
        cudaError_t e_ = cudaGetLastError(); \
        if (e_ != cudaSuccess) return (int)e_; \
    } while (0)
