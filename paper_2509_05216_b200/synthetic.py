"""Synthetic isosurface workloads of BASELINE.json's named shapes, built with
the reference's own dataset recipe (tests/conftest.py:35-44 build_dataset):

* volume: the gyroid sin x cos y + sin y cos z + sin z cos x on an n^3
  lattice with coordinate i*2*pi*periods/(n-1) (volume.gyroid_grid);
* points: extract_isosurface_points (volume.py:229-276) on the GPU
  (volume.py here, bit-exact), seeded subsample to max_points;
* cameras: the reference orbit (inward fibonacci sphere, radius 1.5 x half
  diagonal, 60 deg fov; tests/conftest.py:25-32);
* ground truth: quantize8(raycast_isosurface(...)) (raycast.py:223-262) on the
  GPU, stored as the 8-bit codes a PNG view holds.

gyroid_points is the host (numpy) restatement of the same extraction, used
by bench.py's CPU arm so that no GPU kernel touches the reference arm.
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
                  resolution: int | None = None, log=print, view_ids=None) -> Workload:
    """The named workload on `device`.  view_ids: raycast the GT of only these
    views of the full orbit (images_u8[k] is view view_ids[k]; `cameras`
    still holds every orbit view)."""
    import time
    from .training import init_log_scales
    n, periods, mp, res, nv = CONFIGS[name]
    mp = max_points or mp
    res = resolution or res
    nv = views or nv
    from . import volume as V
    t0 = time.time()
    grid = V.gyroid_grid(n, periods)
    pc = V.extract_isosurface_points(grid, 0.0, max_points=mp, seed=0)
    pos, normals = pc.positions, pc.normals
    t1 = time.time()
    ls = init_log_scales(pos)
    t2 = time.time()
    cams = orbit(n, nv, res)
    data = grid.device_data(device)
    grid = V.VolumeGrid(grid.dims, grid.spacing, grid.origin, data)
    ids = list(range(nv)) if view_ids is None else [int(v) for v in view_ids]
    imgs = torch.empty((len(ids), res, res, 3), dtype=torch.uint8, device=device)
    for k, v in enumerate(ids):
        imgs[k] = V.raycast_isosurface(grid, 0.0, cams[v], codes=True)
    torch.cuda.synchronize()
    t3 = time.time()
    log(f"[workload {name}] {pos.shape[0]} points ({t1 - t0:.1f}s), kNN scales ({t2 - t1:.1f}s), "
        f"{len(ids)} raycast GT views at {res}^2 ({t3 - t2:.1f}s)")
    del grid, data
    return Workload(name, pos, normals, ls, cams, imgs, res)
