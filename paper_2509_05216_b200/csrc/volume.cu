// volume.cu -- dataset generation on the device (sm_100a): isosurface point
// extraction and the first-hit isosurface raycaster that makes the ground
// truth views.
//
//   isg_iso_edges   : edge crossings of one lattice axis, in C order
//                     (volume.py:197-226 _axis_crossings);
//   isg_iso_normals : normalised central-difference gradients at points
//                     (volume.py:108-174 sample_trilinear / gradient_central,
//                     volume.py:270-275);
//   isg_raycast     : raycast_isosurface (raycast.py:19-220), one thread per
//                     pixel, optional quantize8 codes (images.py:9-16).
//
// All arithmetic is float64 in the reference's statement order and this unit
// is compiled with -fmad=false, so every output is bit-identical to the
// numpy / numba reference (tests/test_volume.py pins it).
#include <cub/cub.cuh>

#include "common.cuh"

namespace isg {

struct Grid {
    const double *data;  // (nz, ny, nx), x fastest
    int nx, ny, nz;
    double ox, oy, oz, sx, sy, sz;
};

// _tri (raycast.py:19-69): clamped trilinear sample.  sample_trilinear
// (volume.py:108-143) is the same arithmetic (floor of a clamped non-negative
// coordinate == int truncation).
__device__ __forceinline__ double tri(const Grid &g, double px, double py, double pz) {
    double vx = (px - g.ox) / g.sx;
    double vy = (py - g.oy) / g.sy;
    double vz = (pz - g.oz) / g.sz;
    if (vx < 0.0) vx = 0.0;
    else if (vx > g.nx - 1.0) vx = g.nx - 1.0;
    if (vy < 0.0) vy = 0.0;
    else if (vy > g.ny - 1.0) vy = g.ny - 1.0;
    if (vz < 0.0) vz = 0.0;
    else if (vz > g.nz - 1.0) vz = g.nz - 1.0;
    int x0 = (int)vx, y0 = (int)vy, z0 = (int)vz;
    if (x0 > g.nx - 2) x0 = g.nx - 2;
    if (y0 > g.ny - 2) y0 = g.ny - 2;
    if (z0 > g.nz - 2) z0 = g.nz - 2;
    if (x0 < 0) x0 = 0;
    if (y0 < 0) y0 = 0;
    if (z0 < 0) z0 = 0;
    const double fx = vx - x0, fy = vy - y0, fz = vz - z0;
    const int64_t sy_ = g.nx, sz_ = (int64_t)g.nx * g.ny;
    const double *d = g.data + (int64_t)z0 * sz_ + (int64_t)y0 * sy_ + x0;
    // single-slice axes (n = 1) never reach the +1 corner with a non-zero weight
    const int64_t dx = g.nx > 1 ? 1 : 0, dy = g.ny > 1 ? sy_ : 0, dz = g.nz > 1 ? sz_ : 0;
    const double c000 = d[0], c100 = d[dx], c010 = d[dy], c110 = d[dy + dx];
    const double c001 = d[dz], c101 = d[dz + dx], c011 = d[dz + dy], c111 = d[dz + dy + dx];
    const double c00 = c000 + (c100 - c000) * fx;
    const double c10 = c010 + (c110 - c010) * fx;
    const double c01 = c001 + (c101 - c001) * fx;
    const double c11 = c011 + (c111 - c011) * fx;
    const double c0 = c00 + (c10 - c00) * fy;
    const double c1 = c01 + (c11 - c01) * fy;
    return c0 + (c1 - c0) * fz;
}

// Central difference along one axis with one-sided fallback at the box
// (raycast.py:72-96; gradient_central, volume.py:146-174).
__device__ __forceinline__ double grad_axis(const Grid &g, double px, double py, double pz,
                                            int axis, const double (&wmin)[3],
                                            const double (&wmax)[3]) {
    double h, fh, fl;
    bool lo_ok, hi_ok;
    if (axis == 0) {
        h = g.sx;
        lo_ok = px - h >= wmin[0] - 1e-12;
        hi_ok = px + h <= wmax[0] + 1e-12;
        fh = tri(g, hi_ok ? px + h : px, py, pz);
        fl = tri(g, lo_ok ? px - h : px, py, pz);
    } else if (axis == 1) {
        h = g.sy;
        lo_ok = py - h >= wmin[1] - 1e-12;
        hi_ok = py + h <= wmax[1] + 1e-12;
        fh = tri(g, px, hi_ok ? py + h : py, pz);
        fl = tri(g, px, lo_ok ? py - h : py, pz);
    } else {
        h = g.sz;
        lo_ok = pz - h >= wmin[2] - 1e-12;
        hi_ok = pz + h <= wmax[2] + 1e-12;
        fh = tri(g, px, py, hi_ok ? pz + h : pz);
        fl = tri(g, px, py, lo_ok ? pz - h : pz);
    }
    const double denom = h * ((hi_ok ? 1.0 : 0.0) + (lo_ok ? 1.0 : 0.0));
    if (denom <= 0.0) return 0.0;
    return (fh - fl) / denom;
}

__device__ __forceinline__ void grid_box(const Grid &g, double (&wmin)[3], double (&wmax)[3]) {
    wmin[0] = g.ox;
    wmin[1] = g.oy;
    wmin[2] = g.oz;
    wmax[0] = g.ox + (g.nx - 1.0) * g.sx;
    wmax[1] = g.oy + (g.ny - 1.0) * g.sy;
    wmax[2] = g.oz + (g.nz - 1.0) * g.sz;
}

// ---------------------------------------------------------------- raycast --
__global__ void __launch_bounds__(128) raycast_kernel(Grid g, double iso, Cam cam, double step,
                                                      int refine_steps, double al0, double al1,
                                                      double al2, double bg0, double bg1,
                                                      double bg2, double *__restrict__ out,
                                                      uint8_t *__restrict__ codes) {
    const int px = blockIdx.x * 16 + (threadIdx.x & 15);
    const int py = blockIdx.y * 8 + (threadIdx.x >> 4);
    if (px >= cam.width || py >= cam.height) return;
    double wmin[3], wmax[3];
    grid_box(g, wmin, wmax);
    const double *rot = cam.R, *cp = cam.C;
    double dcx = (px - cam.cx) / cam.fx;
    double dcy = (py - cam.cy) / cam.fy;
    const double inv = 1.0 / sqrt(dcx * dcx + dcy * dcy + 1.0);
    dcx *= inv;
    dcy *= inv;
    const double dcz = inv;
    const double dx = rot[0] * dcx + rot[3] * dcy + rot[6] * dcz;
    const double dy = rot[1] * dcx + rot[4] * dcy + rot[7] * dcz;
    const double dz = rot[2] * dcx + rot[5] * dcy + rot[8] * dcz;
    double t0 = -1e30, t1 = 1e30;
    bool hit_box = true;
    for (int axis = 0; axis < 3; axis++) {
        const double o = cp[axis], d = axis == 0 ? dx : (axis == 1 ? dy : dz);
        const double lo = wmin[axis], hi = wmax[axis];
        if (fabs(d) < 1e-15) {
            if (o < lo || o > hi) {
                hit_box = false;
                break;
            }
        } else {
            double ta = (lo - o) / d, tb = (hi - o) / d;
            if (ta > tb) {
                const double s = ta;
                ta = tb;
                tb = s;
            }
            if (ta > t0) t0 = ta;
            if (tb < t1) t1 = tb;
        }
    }
    double c[3] = {bg0, bg1, bg2};
    bool found = false;
    double t_hit = 0.0;
    if (hit_box && !(t1 < t0)) {
        if (t0 < 0.0) t0 = 0.0;
        double fa = tri(g, cp[0] + t0 * dx, cp[1] + t0 * dy, cp[2] + t0 * dz) - iso;
        double ta = t0, t = t0;
        while (t < t1) {
            t = t + step;
            if (t > t1) t = t1;
            const double fb = tri(g, cp[0] + t * dx, cp[1] + t * dy, cp[2] + t * dz) - iso;
            if (fa * fb < 0.0 || fb == 0.0) {
                double tb_ = t, fa_ = fa, fb_ = fb, ta_ = ta;
                for (int it = 0; it < refine_steps; it++) {
                    const double tm = 0.5 * (ta_ + tb_);
                    const double fm =
                        tri(g, cp[0] + tm * dx, cp[1] + tm * dy, cp[2] + tm * dz) - iso;
                    if (fa_ * fm < 0.0) {
                        tb_ = tm;
                        fb_ = fm;
                    } else {
                        ta_ = tm;
                        fa_ = fm;
                    }
                }
                // close from the final bracket with its linear zero crossing
                if (fb_ != fa_)
                    t_hit = ta_ + (tb_ - ta_) * (-fa_) / (fb_ - fa_);
                else
                    t_hit = 0.5 * (ta_ + tb_);
                found = true;
                break;
            }
            fa = fb;
            ta = t;
            if (t >= t1) break;
        }
    }
    if (found) {
        const double hx = cp[0] + t_hit * dx, hy = cp[1] + t_hit * dy, hz = cp[2] + t_hit * dz;
        const double gx = grad_axis(g, hx, hy, hz, 0, wmin, wmax);
        const double gy = grad_axis(g, hx, hy, hz, 1, wmin, wmax);
        const double gz = grad_axis(g, hx, hy, hz, 2, wmin, wmax);
        const double gn = sqrt(gx * gx + gy * gy + gz * gz);
        double nxv, nyv, nzv;
        if (gn < 1e-12) {
            nxv = 0.0;
            nyv = 0.0;
            nzv = 1.0;
        } else {
            nxv = gx / gn;
            nyv = gy / gn;
            nzv = gz / gn;
        }
        double ndd = nxv * dx + nyv * dy + nzv * dz;
        if (ndd > 0.0) ndd = -ndd;  // normal flipped to face the ray
        double lam = -ndd;
        if (lam < 0.0) lam = 0.0;
        const double al[3] = {al0, al1, al2};
        for (int k = 0; k < 3; k++) {
            double v = al[k] * lam;
            if (v < 0.0) v = 0.0;
            else if (v > 1.0) v = 1.0;
            c[k] = v;
        }
    }
    const int64_t pix = (int64_t)py * cam.width + px;
    if (out) {
        out[3 * pix] = c[0];
        out[3 * pix + 1] = c[1];
        out[3 * pix + 2] = c[2];
    }
    if (codes) {
        // quantize8: rint(clip(v, 0, 1) * 255), ties to even
        for (int k = 0; k < 3; k++)
            codes[3 * pix + k] = (uint8_t)rint(fmin(fmax(c[k], 0.0), 1.0) * 255.0);
    }
}

// ------------------------------------------------------- point extraction --
// Edge domain of one axis on the strided sub-lattice: (ez, ey, ex) edge starts,
// C order.  axis_data: 2 = x edges, 1 = y, 0 = z (volume.py:197-209).
struct Edges {
    const double *data;
    int nx, ny, nz, stride, axis;
    int ex, ey, ez;
    double iso;

    __device__ __forceinline__ void at(int64_t i, int &kx, int &ky, int &kz) const {
        kx = (int)(i % ex);
        const int64_t r = i / ex;
        ky = (int)(r % ey);
        kz = (int)(r / ey);
    }
    __device__ __forceinline__ double val(int kx, int ky, int kz) const {
        return data[((int64_t)kz * stride * ny + (int64_t)ky * stride) * nx + (int64_t)kx * stride];
    }
    __device__ __forceinline__ void ends(int64_t i, double &v0, double &v1) const {
        int kx, ky, kz;
        at(i, kx, ky, kz);
        v0 = val(kx, ky, kz);
        v1 = val(kx + (axis == 2), ky + (axis == 1), kz + (axis == 0));
    }
    __device__ __forceinline__ bool operator()(const int64_t &i) const {
        double v0, v1;
        ends(i, v0, v1);
        return (v0 - iso) * (v1 - iso) < 0.0;
    }
};

inline Edges make_edges(const double *data, int nx, int ny, int nz, int stride, int axis,
                        double iso) {
    Edges e;
    e.data = data;
    e.nx = nx;
    e.ny = ny;
    e.nz = nz;
    e.stride = stride;
    e.axis = axis;
    e.iso = iso;
    const int sx = (nx + stride - 1) / stride, sy = (ny + stride - 1) / stride,
              sz = (nz + stride - 1) / stride;
    e.ex = sx - (axis == 2);
    e.ey = sy - (axis == 1);
    e.ez = sz - (axis == 0);
    return e;
}

// world_min + idx * (stride * spacing), idx[world_axis] += t (volume.py:221-226)
__global__ void edge_points_kernel(Edges e, int64_t n, const int64_t *__restrict__ idx,
                                   double ox, double oy, double oz, double sx, double sy,
                                   double sz, double *__restrict__ pos) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int kx, ky, kz;
    e.at(idx[j], kx, ky, kz);
    double v0, v1;
    e.ends(idx[j], v0, v1);
    const double t = (e.iso - v0) / (v1 - v0);
    double fx = (double)kx, fy = (double)ky, fz = (double)kz;
    if (e.axis == 2) fx += t;
    else if (e.axis == 1) fy += t;
    else fz += t;
    const double st = (double)e.stride;
    pos[3 * j] = ox + fx * (st * sx);
    pos[3 * j + 1] = oy + fy * (st * sy);
    pos[3 * j + 2] = oz + fz * (st * sz);
}

// gradient_central + the normalisation of extract_isosurface_points.
__global__ void iso_normals_kernel(Grid g, int64_t n, const double *__restrict__ pos,
                                   double *__restrict__ nrm) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    double wmin[3], wmax[3];
    grid_box(g, wmin, wmax);
    const double px = pos[3 * j], py = pos[3 * j + 1], pz = pos[3 * j + 2];
    const double gx = grad_axis(g, px, py, pz, 0, wmin, wmax);
    const double gy = grad_axis(g, px, py, pz, 1, wmin, wmax);
    const double gz = grad_axis(g, px, py, pz, 2, wmin, wmax);
    const double norm = sqrt(gx * gx + gy * gy + gz * gz);
    if (norm > 1e-12) {
        nrm[3 * j] = gx / norm;
        nrm[3 * j + 1] = gy / norm;
        nrm[3 * j + 2] = gz / norm;
    } else {
        nrm[3 * j] = 0.0;
        nrm[3 * j + 1] = 0.0;
        nrm[3 * j + 2] = 1.0;
    }
}

inline Grid make_grid(const double *data, const int32_t *dims, const double *spacing,
                      const double *origin) {
    Grid g;
    g.data = data;
    g.nx = dims[0];
    g.ny = dims[1];
    g.nz = dims[2];
    g.sx = spacing[0];
    g.sy = spacing[1];
    g.sz = spacing[2];
    g.ox = origin[0];
    g.oy = origin[1];
    g.oz = origin[2];
    return g;
}

inline bool grid_ok(const int32_t *dims, const double *spacing, const double *origin) {
    return dims && spacing && origin && dims[0] >= 1 && dims[1] >= 1 && dims[2] >= 1 &&
           spacing[0] > 0.0 && spacing[1] > 0.0 && spacing[2] > 0.0;
}

}  // namespace isg

using namespace isg;

extern "C" int isg_raycast(const double *data, const int32_t *dims, const double *spacing,
                           const double *origin, double isovalue, const isg_camera *cam,
                           double step, int32_t refine_steps, const double *albedo,
                           const double *background, double *image, uint8_t *codes,
                           void *stream) {
    if (!data || !grid_ok(dims, spacing, origin) || !cam || !albedo || !background ||
        !(step > 0.0) || refine_steps < 0 || cam->width <= 0 || cam->height <= 0 ||
        (!image && !codes))
        return (int)cudaErrorInvalidValue;
    const Grid g = make_grid(data, dims, spacing, origin);
    dim3 grid((cam->width + 15) / 16, (cam->height + 7) / 8);
    raycast_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(
        g, isovalue, to_cam(*cam), step, refine_steps, albedo[0], albedo[1], albedo[2],
        background[0], background[1], background[2], image, codes);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_iso_edges(void *workspace, size_t *ws_bytes, const double *data,
                             const int32_t *dims, int32_t stride, int32_t axis_data,
                             double isovalue, int64_t *idx_out, int64_t *count, void *stream) {
    if (!ws_bytes || !dims || stride < 1 || axis_data < 0 || axis_data > 2 || dims[0] < 1 ||
        dims[1] < 1 || dims[2] < 1)
        return (int)cudaErrorInvalidValue;
    const Edges e = make_edges(data, dims[0], dims[1], dims[2], stride, axis_data, isovalue);
    const int64_t n = (e.ex > 0 && e.ey > 0 && e.ez > 0) ? (int64_t)e.ex * e.ey * e.ez : 0;
    cub::CountingInputIterator<int64_t> it(0);
    size_t need = 0;
    cudaError_t err = cub::DeviceSelect::If(nullptr, need, it, idx_out, count, n, e,
                                            (cudaStream_t)stream);
    if (err != cudaSuccess) return (int)err;
    if (!workspace) {
        *ws_bytes = need > 0 ? need : 1;
        return 0;
    }
    if (*ws_bytes < need || !data || !idx_out || !count) return (int)cudaErrorInvalidValue;
    if (n == 0) return (int)cudaMemsetAsync(count, 0, sizeof(int64_t), (cudaStream_t)stream);
    return (int)cub::DeviceSelect::If(workspace, *ws_bytes, it, idx_out, count, n, e,
                                      (cudaStream_t)stream);
}

extern "C" int isg_iso_edge_points(const double *data, const int32_t *dims,
                                   const double *spacing, const double *origin, int32_t stride,
                                   int32_t axis_data, double isovalue, int64_t n,
                                   const int64_t *idx, double *positions, void *stream) {
    if (!grid_ok(dims, spacing, origin) || stride < 1 || axis_data < 0 || axis_data > 2 ||
        n < 0 || (n > 0 && (!data || !idx || !positions)))
        return (int)cudaErrorInvalidValue;
    if (n == 0) return 0;
    const Edges e = make_edges(data, dims[0], dims[1], dims[2], stride, axis_data, isovalue);
    edge_points_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
        e, n, idx, origin[0], origin[1], origin[2], spacing[0], spacing[1], spacing[2],
        positions);
    ISG_CHECK_LAUNCH();
    return 0;
}

extern "C" int isg_iso_normals(const double *data, const int32_t *dims, const double *spacing,
                               const double *origin, int64_t n, const double *positions,
                               double *normals, void *stream) {
    if (!grid_ok(dims, spacing, origin) || n < 0 ||
        (n > 0 && (!data || !positions || !normals)))
        return (int)cudaErrorInvalidValue;
    if (n == 0) return 0;
    iso_normals_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
        make_grid(data, dims, spacing, origin), n, positions, normals);
    ISG_CHECK_LAUNCH();
    return 0;
}
