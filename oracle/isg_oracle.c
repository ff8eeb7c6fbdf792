/*
 * isg_oracle.c -- CPU restatement of the reference training-step hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, loads or
 * calls this file.  It is used by tests/ (as the parity checker), by
 * __graft_entry__.smoke() (as the checker of the smoke run) and by bench.py's
 * cpu_baseline / --impl reference leg (as the timed CPU port of the
 * reference).  See oracle/README.md.
 *
 * Every function follows the reference algorithm (isosplat 0.1.0, paths
 * relative to /root/reference/pkg/src/isosplat/) in strict left-to-right
 * float64 arithmetic.  The file MUST be compiled with -ffp-contract=off and
 * linked against glibc libm so that exp/sqrt match what numba emits (numba
 * never contracts to FMA and lowers np.exp to libm exp).  Parity of this
 * restatement against the reference is pinned by tests/golden/ (fixtures
 * produced by importing the reference itself; tests/golden/make_golden.py and
 * make_golden_dist.py), checked by tests/test_oracle_golden.py.
 *
 * Threading: OpenMP over independent units (Gaussians, tiles, image rows),
 * mirroring the reference's worker-thread parallelism.  Results do not
 * depend on the thread count: every output element is produced by exactly
 * one thread in the same sequential order as the reference.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* _kernels.py:15-22 */
#define SH_C0 0.28209479177387814
#define SH_C1 0.4886025119029199
#define NEAR_PLANE 0.01
#define COV_DILATION 0.3
#define ALPHA_CLAMP 0.99
#define T_STOP 1e-4
static const double ALPHA_SKIP = 1.0 / 255.0;

typedef struct {
    double R[9];   /* world->camera rotation, row major */
    double t[3];   /* translation: q = R p + t */
    double C[3];   /* camera centre in world space (-R^T t) */
    double fx, fy, cx, cy;
    int32_t width, height;
} orc_camera;

/* Indices into the intermediate vector produced by project_core; the layout
 * follows the tuple documented at _kernels.py:29-35. */
enum {
    PC_QX = 1, PC_QY, PC_QZ, PC_U, PC_V, PC_CA, PC_CB, PC_CC, PC_DET,
    PC_KA, PC_KB, PC_KC, PC_RAD, PC_OPAC, PC_R, PC_G, PC_B,
    PC_PR, PC_PG, PC_PB, PC_DX, PC_DY, PC_DZ, PC_VLEN,
    PC_NW, PC_NX, PC_NY, PC_NZ, PC_QN, PC_S0, PC_S1, PC_S2,
    PC_R00, PC_R01, PC_R02, PC_R10, PC_R11, PC_R12, PC_R20, PC_R21, PC_R22,
    PC_U00, PC_U01, PC_U02, PC_U10, PC_U11, PC_U12, PC_COUNT
};

/* _kernels.py:26-140 (_project_core).  Returns 1 when valid. */
static int project_core(double px, double py, double pz,
                        double lsx, double lsy, double lsz,
                        double qw, double qx, double qy, double qz,
                        double logit, const double *sh, int degree,
                        const orc_camera *cam, double *o)
{
    const double *rot = cam->R;
    double qcx = rot[0] * px + rot[1] * py + rot[2] * pz + cam->t[0];
    double qcy = rot[3] * px + rot[4] * py + rot[5] * pz + cam->t[1];
    double qcz = rot[6] * px + rot[7] * py + rot[8] * pz + cam->t[2];
    if (qcz <= NEAR_PLANE) return 0;
    double qnorm = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
    if (qnorm < 1e-12) return 0;
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
    double s20 = exp(2.0 * lsx), s21 = exp(2.0 * lsy), s22 = exp(2.0 * lsz);
    double c00 = r00 * s20 * r00 + r01 * s21 * r01 + r02 * s22 * r02;
    double c01 = r00 * s20 * r10 + r01 * s21 * r11 + r02 * s22 * r12;
    double c02 = r00 * s20 * r20 + r01 * s21 * r21 + r02 * s22 * r22;
    double c11 = r10 * s20 * r10 + r11 * s21 * r11 + r12 * s22 * r12;
    double c12 = r10 * s20 * r20 + r11 * s21 * r21 + r12 * s22 * r22;
    double c22 = r20 * s20 * r20 + r21 * s21 * r21 + r22 * s22 * r22;
    double iz = 1.0 / qcz;
    double iz2 = iz * iz;
    double j00 = cam->fx * iz;
    double j02 = -cam->fx * qcx * iz2;
    double j11 = cam->fy * iz;
    double j12 = -cam->fy * qcy * iz2;
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
    if (det <= 0.0) return 0;
    double ka = cc / det, kb = -cb / det, kc = ca / det;
    double mid = 0.5 * (ca + cc);
    double disc = mid * mid - det;
    if (disc < 0.0) disc = 0.0;
    double lam = mid + sqrt(disc);
    double radius = 3.0 * sqrt(lam);
    double u = cam->fx * qcx * iz + cam->cx;
    double v = cam->fy * qcy * iz + cam->cy;
    double opac = 1.0 / (1.0 + exp(-logit));
    double vx = px - cam->C[0], vy = py - cam->C[1], vz = pz - cam->C[2];
    double vlen = sqrt(vx * vx + vy * vy + vz * vz);
    if (vlen < 1e-12) return 0;
    double dx = vx / vlen, dy = vy / vlen, dz = vz / vlen;
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
    /* min(max(x, 0), 1) with Python builtin semantics */
    double cr = pr, cg = pg, cbl = pb;
    if (0.0 > cr) cr = 0.0;
    if (1.0 < cr) cr = 1.0;
    if (0.0 > cg) cg = 0.0;
    if (1.0 < cg) cg = 1.0;
    if (0.0 > cbl) cbl = 0.0;
    if (1.0 < cbl) cbl = 1.0;
    o[PC_QX] = qcx; o[PC_QY] = qcy; o[PC_QZ] = qcz; o[PC_U] = u; o[PC_V] = v;
    o[PC_CA] = ca; o[PC_CB] = cb; o[PC_CC] = cc; o[PC_DET] = det;
    o[PC_KA] = ka; o[PC_KB] = kb; o[PC_KC] = kc; o[PC_RAD] = radius;
    o[PC_OPAC] = opac; o[PC_R] = cr; o[PC_G] = cg; o[PC_B] = cbl;
    o[PC_PR] = pr; o[PC_PG] = pg; o[PC_PB] = pb;
    o[PC_DX] = dx; o[PC_DY] = dy; o[PC_DZ] = dz; o[PC_VLEN] = vlen;
    o[PC_NW] = nqw; o[PC_NX] = nqx; o[PC_NY] = nqy; o[PC_NZ] = nqz; o[PC_QN] = qnorm;
    o[PC_S0] = s20; o[PC_S1] = s21; o[PC_S2] = s22;
    o[PC_R00] = r00; o[PC_R01] = r01; o[PC_R02] = r02;
    o[PC_R10] = r10; o[PC_R11] = r11; o[PC_R12] = r12;
    o[PC_R20] = r20; o[PC_R21] = r21; o[PC_R22] = r22;
    o[PC_U00] = u00; o[PC_U01] = u01; o[PC_U02] = u02;
    o[PC_U10] = u10; o[PC_U11] = u11; o[PC_U12] = u12;
    return 1;
}

/* _kernels.py:144-198 (_project_kernel).  sh is (n, K, 3), K=(degree+1)^2. */
void orc_project(int64_t n, const double *pos, const double *ls, const double *rot,
                 const double *logit, const double *sh, int degree,
                 const orc_camera *cam, int tile_size, int tiles_x, int tiles_y,
                 uint8_t *flag, double *mean2d, double *cov2d, double *conic,
                 double *depth, double *color, double *opacity, int32_t *tiles)
{
    int k = (degree + 1) * (degree + 1);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double o[PC_COUNT];
        double shl[12];
        for (int j = 0; j < 12; j++) shl[j] = 0.0;
        for (int j = 0; j < 3 * k; j++) shl[j] = sh[i * 3 * k + j];
        flag[i] = 0;
        if (!project_core(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2],
                          ls[3 * i], ls[3 * i + 1], ls[3 * i + 2],
                          rot[4 * i], rot[4 * i + 1], rot[4 * i + 2], rot[4 * i + 3],
                          logit[i], shl, degree, cam, o))
            continue;
        double u = o[PC_U], v = o[PC_V], r = o[PC_RAD];
        if (u + r < 0.0 || u - r > cam->width - 1.0 ||
            v + r < 0.0 || v - r > cam->height - 1.0)
            continue;
        int tx0 = (int)floor((u - r) / tile_size);
        int tx1 = (int)floor((u + r) / tile_size);
        int ty0 = (int)floor((v - r) / tile_size);
        int ty1 = (int)floor((v + r) / tile_size);
        if (tx1 < 0 || ty1 < 0 || tx0 >= tiles_x || ty0 >= tiles_y) continue;
        if (tx0 < 0) tx0 = 0;
        if (ty0 < 0) ty0 = 0;
        if (tx1 >= tiles_x) tx1 = tiles_x - 1;
        if (ty1 >= tiles_y) ty1 = tiles_y - 1;
        flag[i] = 1;
        mean2d[2 * i] = u; mean2d[2 * i + 1] = v;
        cov2d[3 * i] = o[PC_CA]; cov2d[3 * i + 1] = o[PC_CB]; cov2d[3 * i + 2] = o[PC_CC];
        conic[3 * i] = o[PC_KA]; conic[3 * i + 1] = o[PC_KB]; conic[3 * i + 2] = o[PC_KC];
        depth[i] = o[PC_QZ];
        color[3 * i] = o[PC_R]; color[3 * i + 1] = o[PC_G]; color[3 * i + 2] = o[PC_B];
        opacity[i] = o[PC_OPAC];
        tiles[4 * i] = tx0; tiles[4 * i + 1] = ty0; tiles[4 * i + 2] = tx1; tiles[4 * i + 3] = ty1;
    }
}

/* _kernels.py:202-211 (_count_tile_entries) */
void orc_count_tile_entries(int64_t m, const int32_t *rects, const int32_t *tile_slot,
                            int tiles_x, int64_t *counts)
{
    for (int64_t i = 0; i < m; i++)
        for (int ty = rects[4 * i + 1]; ty <= rects[4 * i + 3]; ty++)
            for (int tx = rects[4 * i]; tx <= rects[4 * i + 2]; tx++) {
                int32_t slot = tile_slot[(int64_t)ty * tiles_x + tx];
                if (slot >= 0) counts[slot] += 1;
            }
}

/* _kernels.py:215-225 (_fill_tile_entries) */
void orc_fill_tile_entries(int64_t m, const int32_t *rects, const int32_t *tile_slot,
                           int tiles_x, const int64_t *offsets, int64_t *cursor,
                           int32_t *entries)
{
    for (int64_t i = 0; i < m; i++)
        for (int ty = rects[4 * i + 1]; ty <= rects[4 * i + 3]; ty++)
            for (int tx = rects[4 * i]; tx <= rects[4 * i + 2]; tx++) {
                int32_t slot = tile_slot[(int64_t)ty * tiles_x + tx];
                if (slot >= 0) {
                    entries[offsets[slot] + cursor[slot]] = (int32_t)i;
                    cursor[slot] += 1;
                }
            }
}

/* _kernels.py:229-278 (_forward_tiles).  image is (H, W, 3) float64 here; the
 * wrapper casts to the requested dtype exactly as numba's store would.
 * touched may be NULL. */
void orc_forward_tiles(int64_t n_tiles, const int32_t *own_tiles, const int64_t *offsets,
                       const int32_t *entries, const double *mean2d, const double *conic,
                       const double *color, const double *opacity, int tiles_x,
                       int tile_size, int width, int height, const double *bg,
                       double *image, double *t_final, int32_t *n_contrib,
                       int64_t *touched)
{
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t k = 0; k < n_tiles; k++) {
        int tid = own_tiles[k];
        int ty = tid / tiles_x, tx = tid % tiles_x;
        int x0 = tx * tile_size, y0 = ty * tile_size;
        int x1 = x0 + tile_size < width ? x0 + tile_size : width;
        int y1 = y0 + tile_size < height ? y0 + tile_size : height;
        int64_t e0 = offsets[k], e1 = offsets[k + 1];
        for (int py = y0; py < y1; py++)
            for (int px = x0; px < x1; px++) {
                double t = 1.0, cr = 0.0, cg = 0.0, cb = 0.0;
                int32_t count = 0;
                for (int64_t e = e0; e < e1; e++) {
                    int32_t s = entries[e];
                    double d0 = px - mean2d[2 * s];
                    double d1 = py - mean2d[2 * s + 1];
                    double power = (-0.5 * (conic[3 * s] * d0 * d0 + conic[3 * s + 2] * d1 * d1)
                                    - conic[3 * s + 1] * d0 * d1);
                    if (power > 0.0) continue;
                    double g = exp(power);
                    double alpha = opacity[s] * g;
                    if (alpha > ALPHA_CLAMP) alpha = ALPHA_CLAMP;
                    if (alpha < ALPHA_SKIP) continue;
                    double test = t * (1.0 - alpha);
                    if (test < T_STOP) break;
                    cr += color[3 * s] * alpha * t;
                    cg += color[3 * s + 1] * alpha * t;
                    cb += color[3 * s + 2] * alpha * t;
                    t = test;
                    count += 1;
                    if (touched) {
#pragma omp atomic
                        touched[s] += 1;
                    }
                }
                int64_t pix = (int64_t)py * width + px;
                image[3 * pix] = cr + t * bg[0];
                image[3 * pix + 1] = cg + t * bg[1];
                image[3 * pix + 2] = cb + t * bg[2];
                t_final[pix] = t;
                n_contrib[pix] = count;
            }
    }
}

/* _kernels.py:282-374 (_backward_tiles).  Scratch rows align with entries and
 * must be zeroed by the caller (rasterizer.py:231-236). */
void orc_backward_tiles(int64_t n_tiles, const int32_t *own_tiles, const int64_t *offsets,
                        const int32_t *entries, const double *mean2d, const double *conic,
                        const double *color, const double *opacity, int tiles_x,
                        int tile_size, int width, int height, const double *bg,
                        const double *dl, double *scr_dmean, double *scr_dconic,
                        double *scr_dcolor, double *scr_dopac)
{
    int64_t max_seg = 0;
    for (int64_t k = 0; k < n_tiles; k++)
        if (offsets[k + 1] - offsets[k] > max_seg) max_seg = offsets[k + 1] - offsets[k];
#pragma omp parallel
    {
        double *acc_alpha = (double *)malloc(sizeof(double) * (max_seg + 1));
        double *acc_t = (double *)malloc(sizeof(double) * (max_seg + 1));
        double *acc_g = (double *)malloc(sizeof(double) * (max_seg + 1));
        int64_t *acc_e = (int64_t *)malloc(sizeof(int64_t) * (max_seg + 1));
#pragma omp for schedule(dynamic, 1)
        for (int64_t k = 0; k < n_tiles; k++) {
            int tid = own_tiles[k];
            int ty = tid / tiles_x, tx = tid % tiles_x;
            int x0 = tx * tile_size, y0 = ty * tile_size;
            int x1 = x0 + tile_size < width ? x0 + tile_size : width;
            int y1 = y0 + tile_size < height ? y0 + tile_size : height;
            int64_t e0 = offsets[k], e1 = offsets[k + 1];
            for (int py = y0; py < y1; py++)
                for (int px = x0; px < x1; px++) {
                    double t = 1.0;
                    int64_t count = 0;
                    for (int64_t e = e0; e < e1; e++) {
                        int32_t s = entries[e];
                        double d0 = px - mean2d[2 * s];
                        double d1 = py - mean2d[2 * s + 1];
                        double power = (-0.5 * (conic[3 * s] * d0 * d0 + conic[3 * s + 2] * d1 * d1)
                                        - conic[3 * s + 1] * d0 * d1);
                        if (power > 0.0) continue;
                        double g = exp(power);
                        double alpha = opacity[s] * g;
                        if (alpha > ALPHA_CLAMP) alpha = ALPHA_CLAMP;
                        if (alpha < ALPHA_SKIP) continue;
                        double test = t * (1.0 - alpha);
                        if (test < T_STOP) break;
                        acc_e[count] = e;
                        acc_alpha[count] = alpha;
                        acc_t[count] = t;
                        acc_g[count] = g;
                        t = test;
                        count += 1;
                    }
                    int64_t pix = (int64_t)py * width + px;
                    double wr = dl[3 * pix], wg = dl[3 * pix + 1], wb = dl[3 * pix + 2];
                    double sr = t * bg[0], sg = t * bg[1], sb = t * bg[2];
                    for (int64_t i = count - 1; i >= 0; i--) {
                        int64_t e = acc_e[i];
                        int32_t s = entries[e];
                        double alpha = acc_alpha[i], ti = acc_t[i], g = acc_g[i];
                        double at = alpha * ti;
                        scr_dcolor[3 * e] += wr * at;
                        scr_dcolor[3 * e + 1] += wg * at;
                        scr_dcolor[3 * e + 2] += wb * at;
                        double om = 1.0 - alpha;
                        double dalpha = (wr * (color[3 * s] * ti - sr / om)
                                         + wg * (color[3 * s + 1] * ti - sg / om)
                                         + wb * (color[3 * s + 2] * ti - sb / om));
                        sr += color[3 * s] * at;
                        sg += color[3 * s + 1] * at;
                        sb += color[3 * s + 2] * at;
                        if (opacity[s] * g > ALPHA_CLAMP) continue;
                        double dg = dalpha * opacity[s];
                        scr_dopac[e] += dalpha * g;
                        double dpower = dg * g;
                        double d0 = px - mean2d[2 * s];
                        double d1 = py - mean2d[2 * s + 1];
                        scr_dconic[3 * e] += dpower * (-0.5 * d0 * d0);
                        scr_dconic[3 * e + 1] += dpower * (-(d0 * d1));
                        scr_dconic[3 * e + 2] += dpower * (-0.5 * d1 * d1);
                        scr_dmean[2 * e] += dpower * (conic[3 * s] * d0 + conic[3 * s + 1] * d1);
                        scr_dmean[2 * e + 1] += dpower * (conic[3 * s + 1] * d0 + conic[3 * s + 2] * d1);
                    }
                }
        }
        free(acc_alpha); free(acc_t); free(acc_g); free(acc_e);
    }
}

/* _kernels.py:378-394 (_route_mask); mask is (n, workers) uint8, pre-zeroed. */
void orc_route_mask(int64_t n, const int32_t *rects, int tiles_x, int workers, uint8_t *mask)
{
    for (int64_t i = 0; i < n; i++) {
        int x0 = rects[4 * i], y0 = rects[4 * i + 1], x1 = rects[4 * i + 2], y1 = rects[4 * i + 3];
        if (x1 - x0 + 1 >= workers) {
            for (int w = 0; w < workers; w++) mask[i * workers + w] = 1;
            continue;
        }
        for (int ty = y0; ty <= y1; ty++)
            for (int tx = x0; tx <= x1; tx++)
                mask[i * workers + ((int64_t)ty * tiles_x + tx) % workers] = 1;
    }
}

/* _kernels.py:398-411 (_reduce_scratch).  Accumulators pre-zeroed. */
void orc_reduce_scratch(int64_t e_count, const int32_t *entries, const double *scr_dmean,
                        const double *scr_dconic, const double *scr_dcolor,
                        const double *scr_dopac, double *acc_dmean, double *acc_dconic,
                        double *acc_dcolor, double *acc_dopac)
{
    for (int64_t e = 0; e < e_count; e++) {
        int32_t s = entries[e];
        acc_dmean[2 * s] += scr_dmean[2 * e];
        acc_dmean[2 * s + 1] += scr_dmean[2 * e + 1];
        acc_dconic[3 * s] += scr_dconic[3 * e];
        acc_dconic[3 * s + 1] += scr_dconic[3 * e + 1];
        acc_dconic[3 * s + 2] += scr_dconic[3 * e + 2];
        acc_dcolor[3 * s] += scr_dcolor[3 * e];
        acc_dcolor[3 * s + 1] += scr_dcolor[3 * e + 1];
        acc_dcolor[3 * s + 2] += scr_dcolor[3 * e + 2];
        acc_dopac[s] += scr_dopac[e];
    }
}

/* _kernels.py:415-634 (_chain_kernel).  Outputs pre-zeroed, float64,
 * out_dsh is (n, K, 3). */
void orc_chain(int64_t n, const double *pos, const double *ls, const double *rotq,
               const double *logit, const double *sh, int degree, const orc_camera *cam,
               const uint8_t *flags, const double *acc_dmean, const double *acc_dconic,
               const double *acc_dcolor, const double *acc_dopac, double *out_dpos,
               double *out_dls, double *out_drot, double *out_dlogit, double *out_dsh)
{
    int k = (degree + 1) * (degree + 1);
    const double *rot = cam->R;
    double fx = cam->fx, fy = cam->fy;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        if (flags[i] == 0) continue;
        double o[PC_COUNT];
        double shl[12];
        for (int j = 0; j < 12; j++) shl[j] = 0.0;
        for (int j = 0; j < 3 * k; j++) shl[j] = sh[i * 3 * k + j];
        if (!project_core(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2],
                          ls[3 * i], ls[3 * i + 1], ls[3 * i + 2],
                          rotq[4 * i], rotq[4 * i + 1], rotq[4 * i + 2], rotq[4 * i + 3],
                          logit[i], shl, degree, cam, o))
            continue;
        double qcx = o[PC_QX], qcy = o[PC_QY], qcz = o[PC_QZ];
        double con_a = o[PC_KA], con_b = o[PC_KB], con_c = o[PC_KC];
        double opac = o[PC_OPAC];
        double pre_r = o[PC_PR], pre_g = o[PC_PG], pre_b = o[PC_PB];
        double dirx = o[PC_DX], diry = o[PC_DY], dirz = o[PC_DZ], vlen = o[PC_VLEN];
        double nqw = o[PC_NW], nqx = o[PC_NX], nqy = o[PC_NY], nqz = o[PC_NZ], qnorm = o[PC_QN];
        double s20 = o[PC_S0], s21 = o[PC_S1], s22 = o[PC_S2];
        double r00 = o[PC_R00], r01 = o[PC_R01], r02 = o[PC_R02];
        double r10 = o[PC_R10], r11 = o[PC_R11], r12 = o[PC_R12];
        double r20 = o[PC_R20], r21 = o[PC_R21], r22 = o[PC_R22];
        double u00 = o[PC_U00], u01 = o[PC_U01], u02 = o[PC_U02];
        double u10 = o[PC_U10], u11 = o[PC_U11], u12 = o[PC_U12];
        double du = acc_dmean[2 * i], dv = acc_dmean[2 * i + 1];
        double dca = acc_dconic[3 * i], dcb = acc_dconic[3 * i + 1], dcc = acc_dconic[3 * i + 2];
        double dcr = acc_dcolor[3 * i], dcg = acc_dcolor[3 * i + 1], dcb_col = acc_dcolor[3 * i + 2];
        double dop = acc_dopac[i];
        const double *shi = shl;
        double *dsh = out_dsh + i * 3 * k;

        if (pre_r < 0.0 || pre_r > 1.0) dcr = 0.0;
        if (pre_g < 0.0 || pre_g > 1.0) dcg = 0.0;
        if (pre_b < 0.0 || pre_b > 1.0) dcb_col = 0.0;
        dsh[0] += dcr * SH_C0;
        dsh[1] += dcg * SH_C0;
        dsh[2] += dcb_col * SH_C0;
        double ddirx = 0.0, ddiry = 0.0, ddirz = 0.0;
        if (degree >= 1) {
            dsh[3] += dcr * (-SH_C1) * diry;
            dsh[4] += dcg * (-SH_C1) * diry;
            dsh[5] += dcb_col * (-SH_C1) * diry;
            dsh[6] += dcr * SH_C1 * dirz;
            dsh[7] += dcg * SH_C1 * dirz;
            dsh[8] += dcb_col * SH_C1 * dirz;
            dsh[9] += dcr * (-SH_C1) * dirx;
            dsh[10] += dcg * (-SH_C1) * dirx;
            dsh[11] += dcb_col * (-SH_C1) * dirx;
            ddirx = (-SH_C1) * (dcr * shi[9] + dcg * shi[10] + dcb_col * shi[11]);
            ddiry = (-SH_C1) * (dcr * shi[3] + dcg * shi[4] + dcb_col * shi[5]);
            ddirz = SH_C1 * (dcr * shi[6] + dcg * shi[7] + dcb_col * shi[8]);
        }
        double dot = dirx * ddirx + diry * ddiry + dirz * ddirz;
        double dpx = (ddirx - dirx * dot) / vlen;
        double dpy = (ddiry - diry * dot) / vlen;
        double dpz = (ddirz - dirz * dot) / vlen;

        out_dlogit[i] += dop * opac * (1.0 - opac);

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
        double gq_z = (du * (-fx * qcx * iz2) + dv * (-fy * qcy * iz2)
                       + gj00 * (-fx * iz2) + gj02 * (2.0 * fx * qcx * iz3)
                       + gj11 * (-fy * iz2) + gj12 * (2.0 * fy * qcy * iz3));
        dpx += rot[0] * gq_x + rot[3] * gq_y + rot[6] * gq_z;
        dpy += rot[1] * gq_x + rot[4] * gq_y + rot[7] * gq_z;
        dpz += rot[2] * gq_x + rot[5] * gq_y + rot[8] * gq_z;
        out_dpos[3 * i] += dpx;
        out_dpos[3 * i + 1] += dpy;
        out_dpos[3 * i + 2] += dpz;

        double dm0 = (r00 * (gs00 * r00 + gs01 * r10 + gs02 * r20)
                      + r10 * (gs10 * r00 + gs11 * r10 + gs12 * r20)
                      + r20 * (gs20 * r00 + gs21 * r10 + gs22 * r20));
        double dm1 = (r01 * (gs00 * r01 + gs01 * r11 + gs02 * r21)
                      + r11 * (gs10 * r01 + gs11 * r11 + gs12 * r21)
                      + r21 * (gs20 * r01 + gs21 * r11 + gs22 * r21));
        double dm2 = (r02 * (gs00 * r02 + gs01 * r12 + gs02 * r22)
                      + r12 * (gs10 * r02 + gs11 * r12 + gs12 * r22)
                      + r22 * (gs20 * r02 + gs21 * r12 + gs22 * r22));
        out_dls[3 * i] += dm0 * 2.0 * s20;
        out_dls[3 * i + 1] += dm1 * 2.0 * s21;
        out_dls[3 * i + 2] += dm2 * 2.0 * s22;

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

        double dnw = 2.0 * (gr01 * (-nqz) + gr02 * nqy + gr10 * nqz
                            + gr12 * (-nqx) + gr20 * (-nqy) + gr21 * nqx);
        double dnx = 2.0 * (gr01 * nqy + gr02 * nqz + gr10 * nqy
                            + gr11 * (-2.0 * nqx) + gr12 * (-nqw)
                            + gr20 * nqz + gr21 * nqw + gr22 * (-2.0 * nqx));
        double dny = 2.0 * (gr00 * (-2.0 * nqy) + gr01 * nqx + gr02 * nqw
                            + gr10 * nqx + gr12 * nqz
                            + gr20 * (-nqw) + gr21 * nqz + gr22 * (-2.0 * nqy));
        double dnz = 2.0 * (gr00 * (-2.0 * nqz) + gr01 * (-nqw) + gr02 * nqx
                            + gr10 * nqw + gr11 * (-2.0 * nqz) + gr12 * nqy
                            + gr20 * nqx + gr21 * nqy);
        double ndot = nqw * dnw + nqx * dnx + nqy * dny + nqz * dnz;
        out_drot[4 * i] += (dnw - nqw * ndot) / qnorm;
        out_drot[4 * i + 1] += (dnx - nqx * ndot) / qnorm;
        out_drot[4 * i + 2] += (dny - nqy * ndot) / qnorm;
        out_drot[4 * i + 3] += (dnz - nqz * ndot) / qnorm;
    }
}

/* ---------------------------------------------------------------- loss --- */

/* metrics.py:17-24: the normalised 11-tap Gaussian (sigma 1.5) exactly as the
 * reference computes it (numpy SIMD exp, then w / w.sum()); values pinned from
 * the reference in this container (tests/golden/make_golden.py prints them). */
static const double W1D[11] = {
    0x1.0d956b52a1d70p-10, 0x1.f1fe01ae5a5b8p-8, 0x1.26eb175d83f67p-5,
    0x1.bff0fe8e98418p-4, 0x1.b43c3f52b19f2p-3, 0x1.106560aa892c0p-2,
    0x1.b43c3f52b19f2p-3, 0x1.bff0fe8e98418p-4, 0x1.26eb175d83f67p-5,
    0x1.f1fe01ae5a5b8p-8, 0x1.0d956b52a1d70p-10};

/* numpy's pairwise summation for contiguous float64 add.reduce
 * (numpy/_core/src/umath/loops_utils.h.src, PW_BLOCKSIZE 128), which is what
 * np.sum / np.mean in metrics.py:157, 173 use. */
static double pairwise_sum(const double *a, int64_t n)
{
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
    }
}

/* metrics.py:27-59: valid correlation, rows then columns. x is (h, w). */
static void corr_valid(const double *x, int h, int w, double *tmp, double *out)
{
    int wc = w - 10, hc = h - 10;
    for (int r = 0; r < h; r++)
        for (int c = 0; c < wc; c++) {
            double acc = 0.0;
            for (int i = 0; i < 11; i++) acc += W1D[i] * x[(int64_t)r * w + c + i];
            tmp[(int64_t)r * wc + c] = acc;
        }
    for (int r = 0; r < hc; r++)
        for (int c = 0; c < wc; c++) {
            double acc = 0.0;
            for (int i = 0; i < 11; i++) acc += W1D[i] * tmp[(int64_t)(r + i) * wc + c];
            out[(int64_t)r * wc + c] = acc;
        }
}

/* metrics.py:62-72: adjoint of corr_valid for an (h-10, w-10) field. */
static void corr_adjoint(const double *field, int h, int w, double *canvas,
                         double *tmp, double *out)
{
    int hp = h + 10, wp = w + 10, hc = h - 10, wc = w - 10;
    memset(canvas, 0, sizeof(double) * (size_t)hp * wp);
    for (int r = 0; r < hc; r++)
        for (int c = 0; c < wc; c++)
            canvas[(int64_t)(r + 10) * wp + (c + 10)] = field[(int64_t)r * wc + c];
    corr_valid(canvas, hp, wp, tmp, out);
}

/* metrics.py:135-189 (loss_l1_dssim).  img/ref are (h, w, 3) float64; grad is
 * (h, w, 3) float64 (the wrapper casts to the image dtype). */
double orc_loss_l1_dssim(int h, int w, const double *img, const double *ref,
                         double lam, double *grad)
{
    int64_t npx = (int64_t)h * w;
    int64_t n_pix = npx * 3;
    int hc = h - 10, wc = w - 10;
    int64_t nc = (int64_t)hc * wc;
    double *absd = (double *)malloc(sizeof(double) * n_pix);
    for (int64_t i = 0; i < n_pix; i++) {
        double d = img[i] - ref[i];
        absd[i] = fabs(d);
        double sg = d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0);
        grad[i] = sg * ((1.0 - lam) / (double)n_pix);
    }
    double l1 = pairwise_sum(absd, n_pix) / (double)n_pix;
    free(absd);
    double n_centers = 3.0 * (double)hc * (double)wc;
    double gscale = -lam / n_centers;
    double C1 = pow(0.01, 2.0), C2 = pow(0.03, 2.0);
    double ssim_sum = 0.0;

    size_t big = (size_t)(h + 10) * (w + 10);
    double *x = malloc(sizeof(double) * npx), *y = malloc(sizeof(double) * npx);
    double *xx = malloc(sizeof(double) * npx), *yy = malloc(sizeof(double) * npx);
    double *xy = malloc(sizeof(double) * npx);
    double *tmp = malloc(sizeof(double) * big);
    double *canvas = malloc(sizeof(double) * big);
    double *mux = malloc(sizeof(double) * nc), *muy = malloc(sizeof(double) * nc);
    double *mxx = malloc(sizeof(double) * nc), *myy = malloc(sizeof(double) * nc);
    double *mxy = malloc(sizeof(double) * nc), *pq = malloc(sizeof(double) * nc);
    double *f0 = malloc(sizeof(double) * nc), *f1 = malloc(sizeof(double) * nc);
    double *f2 = malloc(sizeof(double) * nc);
    double *g0 = malloc(sizeof(double) * npx), *g1 = malloc(sizeof(double) * npx);
    double *g2 = malloc(sizeof(double) * npx);
    for (int c = 0; c < 3; c++) {
        for (int64_t i = 0; i < npx; i++) {
            x[i] = img[3 * i + c];
            y[i] = ref[3 * i + c];
            xx[i] = x[i] * x[i];
            yy[i] = y[i] * y[i];
            xy[i] = x[i] * y[i];
        }
        corr_valid(x, h, w, tmp, mux);
        corr_valid(y, h, w, tmp, muy);
        corr_valid(xx, h, w, tmp, mxx);
        corr_valid(yy, h, w, tmp, myy);
        corr_valid(xy, h, w, tmp, mxy);
        for (int64_t i = 0; i < nc; i++) {
            double mx = mux[i], my = muy[i];
            double var_x = mxx[i] - mx * mx;
            double var_y = myy[i] - my * my;
            double cov = mxy[i] - mx * my;
            double a1 = 2.0 * mx * my + C1;
            double b1 = mx * mx + my * my + C1;
            double a2 = 2.0 * cov + C2;
            double b2 = var_x + var_y + C2;
            double p = a1 / b1, q = a2 / b2;
            pq[i] = p * q;
            double dp_dmux = (2.0 * my * b1 - 2.0 * mx * a1) / (b1 * b1);
            double d_mu = q * dp_dmux;
            double d_sigma = -((p * q) / b2);
            double d_xy = (2.0 * p) / b2;
            double ff1 = 2.0 * d_sigma;
            double ff2 = d_xy;
            f0[i] = d_mu - ff1 * mx - ff2 * my;
            f1[i] = ff1;
            f2[i] = ff2;
        }
        ssim_sum += pairwise_sum(pq, nc);
        corr_adjoint(f0, h, w, canvas, tmp, g0);
        corr_adjoint(f1, h, w, canvas, tmp, g1);
        corr_adjoint(f2, h, w, canvas, tmp, g2);
        for (int64_t i = 0; i < npx; i++) {
            double g = g0[i] + x[i] * g1[i] + y[i] * g2[i];
            grad[3 * i + c] += gscale * g;
        }
    }
    free(x); free(y); free(xx); free(yy); free(xy); free(tmp); free(canvas);
    free(mux); free(muy); free(mxx); free(myy); free(mxy); free(pq);
    free(f0); free(f1); free(f2); free(g0); free(g1); free(g2);
    double ssim_mean = ssim_sum / n_centers;
    return (1.0 - lam) * l1 + lam * (1.0 - ssim_mean);
}

/* metrics.py:87-132 (ssim via _ssim_maps): mean SSIM over valid centres,
 * averaged over channels.  img/ref (h, w, nch) float64. */
double orc_ssim(int h, int w, int nch, const double *img, const double *ref)
{
    int64_t npx = (int64_t)h * w;
    int hc = h - 10, wc = w - 10;
    int64_t nc = (int64_t)hc * wc;
    double C1 = pow(0.01, 2.0), C2 = pow(0.03, 2.0);
    size_t big = (size_t)h * w;
    double *x = malloc(sizeof(double) * npx), *y = malloc(sizeof(double) * npx);
    double *xx = malloc(sizeof(double) * npx), *yy = malloc(sizeof(double) * npx);
    double *xy = malloc(sizeof(double) * npx);
    double *tmp = malloc(sizeof(double) * big);
    double *maps = malloc(sizeof(double) * nc * nch);
    double *mux = malloc(sizeof(double) * nc), *muy = malloc(sizeof(double) * nc);
    double *mxx = malloc(sizeof(double) * nc), *myy = malloc(sizeof(double) * nc);
    double *mxy = malloc(sizeof(double) * nc);
    for (int c = 0; c < nch; c++) {
        for (int64_t i = 0; i < npx; i++) {
            x[i] = img[nch * i + c];
            y[i] = ref[nch * i + c];
            xx[i] = x[i] * x[i];
            yy[i] = y[i] * y[i];
            xy[i] = x[i] * y[i];
        }
        corr_valid(x, h, w, tmp, mux);
        corr_valid(y, h, w, tmp, muy);
        corr_valid(xx, h, w, tmp, mxx);
        corr_valid(yy, h, w, tmp, myy);
        corr_valid(xy, h, w, tmp, mxy);
        for (int64_t i = 0; i < nc; i++) {
            double mx = mux[i], my = muy[i];
            double var_x = mxx[i] - mx * mx;
            double var_y = myy[i] - my * my;
            double cov = mxy[i] - mx * my;
            double a1 = 2.0 * mx * my + C1;
            double b1 = mx * mx + my * my + C1;
            double a2 = 2.0 * cov + C2;
            double b2 = var_x + var_y + C2;
            maps[c * nc + i] = (a1 / b1) * (a2 / b2);
        }
    }
    double s = pairwise_sum(maps, nc * nch) / (double)(nc * nch);
    free(x); free(y); free(xx); free(yy); free(xy); free(tmp); free(maps);
    free(mux); free(muy); free(mxx); free(myy); free(mxy);
    return s;
}

/* ---------------------------------------------------------------- adam --- */

/* optim.py:20-56 for float32 storage.  numpy demotes the Python-float
 * scalars to float32 before each elementwise op (weak scalars), so every
 * constant arrives here already rounded to float32 by the wrapper:
 * b1, omb1 = f32(1 - beta1), b2, omb2 = f32(1 - beta2), bc1, bc2, lr, eps. */
void orc_adam_f32(int64_t n, float *p, const float *g, float *m, float *v,
                  float b1, float omb1, float b2, float omb2, float bc1, float bc2,
                  float lr, float eps)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        float gi = g[i];
        float mi = m[i] * b1;
        mi = mi + omb1 * gi;
        float vi = v[i] * b2;
        float gg = gi * gi;
        vi = vi + omb2 * gg;
        float mhat = mi / bc1;
        float vhat = vi / bc2;
        float den = sqrtf(vhat) + eps;
        float step = (lr * mhat) / den;
        p[i] = p[i] - step;
        m[i] = mi;
        v[i] = vi;
    }
}

/* optim.py:20-56 for float64 storage. */
void orc_adam_f64(int64_t n, double *p, const double *g, double *m, double *v,
                  double b1, double omb1, double b2, double omb2, double bc1, double bc2,
                  double lr, double eps)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double gi = g[i];
        double mi = m[i] * b1;
        mi = mi + omb1 * gi;
        double vi = v[i] * b2;
        double gg = gi * gi;
        vi = vi + omb2 * gg;
        double mhat = mi / bc1;
        double vhat = vi / bc2;
        double den = sqrt(vhat) + eps;
        double step = (lr * mhat) / den;
        p[i] = p[i] - step;
        m[i] = mi;
        v[i] = vi;
    }
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
