"""Synthetic isosurface workloads of BASELINE.json's named shapes.

Dataset generation is outside the hot path (volume.py,
raycast.py are out of scope), so this module only builds inputs of the right
shape for bench.py and the tests:

* points: edge crossings of a gyroid field sin x cos y + sin y cos z +
  sin z cos x on an n^3 lattice with coordinate i*2*pi*periods/(n-1), the
  reference's extract_isosurface_points recipe (volume.py:229-276: x, then y,
  then z edges in C order, seeded subsample re-sorted into extraction order);
* cameras: the reference orbit (inward fibonacci sphere, radius 1.5 x half
  diagonal, 60 deg fov; tests/conftest.py:25-32);
* ground truth: NOT the reference's raycaster (2.4 s per 2K view on a CPU
  core).  Each view is rendered by this package's forward rasteriser from a
  target cloud (opacity 0.9, headlight-like view-dependent albedo shading
  from the analytic normals) and stored as 8-bit codes like the reference's
  PNG views.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from .camera import OrbitSpec, make_orbit

CONFIGS = {
    # name: (lattice n, periods, max_points, resolution, views)
    "config1": None,  # sphere, CPU-runnable case: tests/golden/config1.npz
    "config2": (256, 3.5, 1_000_000, 1024, 448),
    "config3": (256, 13.0, 4_000_000, 2048, 448),
    "config4": (512, 16.0, 18_000_000, 2048, 448),
}


def gyroid_points(n: int, periods: float, max_points: int | None, seed: int = 0):
    """Isosurface (iso 0) edge crossings of the gyroid lattice, in world units
    (spacing 1, origin 0).  Returns (positions f64 (N,3), normals f64 (N,3))."""
    s = 2.0 * math.pi * periods / (n - 1)
    ax = np.arange(n, dtype=np.float64) * s
    sx, cx = np.sin(ax), np.cos(ax)
    # data[z, y, x] = sin x cos y + sin y cos z + sin z cos x
    data = (sx[None, None, :] * cx[None, :, None] + sx[None, :, None] * cx[:, None, None]
            + sx[:, None, None] * cx[None, None, :])
    parts = []
    for axis_data in (2, 1, 0):  # x, then y, then z edges
        lo = [slice(None)] * 3
        hi = [slice(None)] * 3
        lo[axis_data] = slice(0, -1)
        hi[axis_data] = slice(1, None)
        v0 = data[tuple(lo)]
        v1 = data[tuple(hi)]
        kz, ky, kx = np.nonzero(v0 * v1 < 0.0)
        a, b = v0[kz, ky, kx], v1[kz, ky, kx]
        t = (0.0 - a) / (b - a)
        idx = np.stack([kx, ky, kz], axis=1).astype(np.float64)
        idx[:, 2 - axis_data] += t
        parts.append(idx)
        del v0, v1, kz, ky, kx, a, b, t
    pos = np.concatenate(parts, axis=0)
    del data, parts
    if max_points is not None and pos.shape[0] > max_points:
        rng = np.random.default_rng(seed)
        keep = np.sort(rng.choice(pos.shape[0], size=max_points, replace=False))
        pos = pos[keep]
    # analytic gradient of the field (world units)
    x, y, z = (pos[:, 0] * s, pos[:, 1] * s, pos[:, 2] * s)
    g = np.stack([np.cos(x) * np.cos(y) - np.sin(z) * np.sin(x),
                  -np.sin(x) * np.sin(y) + np.cos(y) * np.cos(z),
                  -np.sin(y) * np.sin(z) + np.cos(z) * np.cos(x)], axis=1)
    nrm = np.linalg.norm(g, axis=1, keepdims=True)
    normals = np.where(nrm > 1e-12, g / np.maximum(nrm, 1e-12), np.array([[0.0, 0.0, 1.0]]))
    return pos, normals


def orbit(n: int, count: int, resolution: int):
    lo = np.zeros(3)
    hi = np.full(3, float(n - 1))
    center = tuple((lo + hi) / 2.0)
    radius = 1.5 * float(np.linalg.norm(hi - lo) / 2.0)
    return make_orbit(OrbitSpec(count=count, center=center, radius=radius,
                                width=resolution, height=resolution))


def target_cloud(points: np.ndarray, normals: np.ndarray, log_scales: np.ndarray, device,
                 albedo=(0.87, 0.80, 0.66)):
    """The ground-truth generator cloud: opacity 0.9 and colour
    albedo * (0.55 + 0.4 n.d) expressed exactly in SH degree 1."""
    from .gaussians import GaussianCloud
    n = points.shape[0]
    c0, c1 = 0.28209479177387814, 0.4886025119029199
    a = np.asarray(albedo)
    sh = np.zeros((n, 4, 3))
    sh[:, 0, :] = (a[None, :] * 0.55 - 0.5) / c0
    k = 0.4 * a[None, :] / c1
    sh[:, 1, :] = -k * normals[:, 1:2]
    sh[:, 2, :] = k * normals[:, 2:3]
    sh[:, 3, :] = -k * normals[:, 0:1]
    rot = np.zeros((n, 4), dtype=np.float32)
    rot[:, 0] = 1.0
    f = lambda v: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).to(device)
    return GaussianCloud(positions=f(points), log_scales=f(log_scales), rotations=f(rot),
                         opacity_logits=f(np.full(n, math.log(0.9 / 0.1))), sh_coeffs=f(sh),
                         degree=1)


@dataclass
class Workload:
    name: str
    points: np.ndarray
    normals: np.ndarray
    log_scales: np.ndarray
    cameras: list
    images_u8: torch.Tensor  # (V, H, W, 3) uint8 on the device
    resolution: int


def make_workload(name: str, device, views: int | None = None, max_points: int | None = None,
                  resolution: int | None = None, log=print) -> Workload:
    import time
    from .engine import Rasterizer
    from .training import init_log_scales
    n, periods, mp, res, nv = CONFIGS[name]
    mp = max_points or mp
    res = resolution or res
    nv = views or nv
    t0 = time.time()
    pos, normals = gyroid_points(n, periods, mp)
    t1 = time.time()
    ls = init_log_scales(pos)
    t2 = time.time()
    cams = orbit(n, nv, res)
    tgt = target_cloud(pos, normals, ls, device)
    r = Rasterizer(tgt.count, res, res, device)
    imgs = torch.empty((nv, res, res, 3), dtype=torch.uint8, device=device)
    for v, cam in enumerate(cams):
        r.forward(tgt, cam)
        imgs[v] = torch.round(torch.clamp(r.image, 0.0, 1.0) * 255.0).to(torch.uint8)
    torch.cuda.synchronize()
    t3 = time.time()
    log(f"[workload {name}] {pos.shape[0]} points ({t1 - t0:.1f}s), kNN scales ({t2 - t1:.1f}s), "
        f"{nv} GT views at {res}^2 ({t3 - t2:.1f}s)")
    del r, tgt
    return Workload(name, pos, normals, ls, cams, imgs, res)
