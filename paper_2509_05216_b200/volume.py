"""Dataset generation on the device: isosurface points and ground-truth views.

Mirrors the reference's volume.py / raycast.py API (VolumeGrid,
extract_isosurface_points, gradient_central, raycast_isosurface,
quantize8) over libisogs (isg_iso_edges / isg_iso_edge_points /
isg_iso_normals / isg_raycast).  Every output is bit-identical to the
reference (float64, reference statement order, no FMA contraction;
tests/test_volume.py against tests/golden/volume.npz).  The seeded
subsample of extract_isosurface_points draws its indices with numpy on the
host exactly as the reference does (volume.py:261-264).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .training import PointCloud

DEFAULT_ALBEDO = (0.87, 0.80, 0.66)  # raycast.py:15
DEFAULT_BACKGROUND = (1.0, 1.0, 1.0)  # raycast.py:16


@dataclass(frozen=True)
class VolumeGrid:
    """volume.py:25-62.  data is float64 (nz, ny, nx), x fastest (numpy or a
    torch tensor); dims = (nx, ny, nz)."""

    dims: tuple
    spacing: tuple
    origin: tuple
    data: object

    def __post_init__(self) -> None:
        nx, ny, nz = self.dims
        if min(nx, ny, nz) < 1:
            raise ValueError(f"dims must be positive, got {self.dims}")
        if any(s <= 0 for s in self.spacing):
            raise ValueError(f"spacing must be positive, got {self.spacing}")
        if tuple(self.data.shape) != (nz, ny, nx):
            raise ValueError(f"data shape {tuple(self.data.shape)} does not match dims "
                             f"{self.dims} (expected {(nz, ny, nx)})")

    @property
    def world_min(self) -> np.ndarray:
        return np.asarray(self.origin, dtype=np.float64)

    @property
    def world_max(self) -> np.ndarray:
        d = np.asarray(self.dims, dtype=np.float64) - 1.0
        return self.world_min + d * np.asarray(self.spacing, dtype=np.float64)

    @property
    def value_range(self) -> tuple[float, float]:
        d = self.data
        if isinstance(d, torch.Tensor):
            return float(d.min()), float(d.max())
        return float(np.min(d)), float(np.max(d))

    def device_data(self, dev) -> torch.Tensor:
        d = self.data
        if isinstance(d, torch.Tensor):
            d = d.to(device=dev, dtype=torch.float64)
        else:
            d = torch.from_numpy(np.ascontiguousarray(d, dtype=np.float64)).to(dev)
        return d.contiguous()


def _grid_args(grid: VolumeGrid):
    dims = (ctypes.c_int32 * 3)(*[int(v) for v in grid.dims])
    sp = (ctypes.c_double * 3)(*[float(v) for v in grid.spacing])
    org = (ctypes.c_double * 3)(*[float(v) for v in grid.origin])
    return dims, sp, org


def _cp(a) -> ctypes.c_void_p:
    return ctypes.cast(a, ctypes.c_void_p)


def extract_isosurface_points(grid: VolumeGrid, isovalue: float, stride: int = 1,
                              max_points: int | None = None, seed: int = 0) -> PointCloud:
    """volume.py:229-276: crossings on x, then y, then z edges (C order each),
    seeded subsample re-sorted into extraction order, unit normals from
    central differences ((0, 0, 1) for a zero gradient).  float64 numpy out."""
    if stride < 1:
        raise ValueError(f"stride must be >= 1, got {stride}")
    lo, hi = grid.value_range
    empty = PointCloud(positions=np.empty((0, 3)), normals=np.empty((0, 3)))
    if not (lo < isovalue < hi):
        return empty
    dev = L.require_cuda()
    lib = L.lib()
    data = grid.device_data(dev)
    dims, sp, org = _grid_args(grid)
    nx, ny, nz = grid.dims
    sub = [(n + stride - 1) // stride for n in (nx, ny, nz)]
    parts = []
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    for axis_data in (2, 1, 0):
        e = list(sub)
        e[2 - axis_data] -= 1
        n_edges = max(e[0], 0) * max(e[1], 0) * max(e[2], 0)
        if n_edges == 0:
            continue
        idx = torch.empty(n_edges, dtype=torch.int64, device=dev)
        sz = ctypes.c_size_t(0)
        L.check(lib.isg_iso_edges(None, ctypes.byref(sz), None, _cp(dims), stride, axis_data,
                                  float(isovalue), None, None, None), "isg_iso_edges (size)")
        ws = torch.empty(max(sz.value, 1), dtype=torch.uint8, device=dev)
        sz = ctypes.c_size_t(ws.numel())
        L.check(lib.isg_iso_edges(L.ptr(ws), ctypes.byref(sz), L.ptr(data), _cp(dims), stride,
                                  axis_data, float(isovalue), L.ptr(idx), L.ptr(count),
                                  L.stream_ptr()), "isg_iso_edges")
        n = int(count.item())
        if n == 0:
            continue
        pos = torch.empty((n, 3), dtype=torch.float64, device=dev)
        L.check(lib.isg_iso_edge_points(L.ptr(data), _cp(dims), _cp(sp), _cp(org), stride,
                                        axis_data, float(isovalue), n, L.ptr(idx), L.ptr(pos),
                                        L.stream_ptr()), "isg_iso_edge_points")
        parts.append(pos)
        del idx, ws
    if not parts:
        return empty
    positions = torch.cat(parts)
    if max_points is not None and positions.shape[0] > max_points:
        rng = np.random.default_rng(seed)
        keep = np.sort(rng.choice(positions.shape[0], size=max_points, replace=False))
        positions = positions[torch.from_numpy(keep).to(dev)].contiguous()
    n = positions.shape[0]
    normals = torch.empty_like(positions)
    L.check(lib.isg_iso_normals(L.ptr(data), _cp(dims), _cp(sp), _cp(org), n, L.ptr(positions),
                                L.ptr(normals), L.stream_ptr()), "isg_iso_normals")
    return PointCloud(positions=positions.cpu().numpy(), normals=normals.cpu().numpy())


def raycast_isosurface(grid: VolumeGrid, isovalue: float, cam, albedo=DEFAULT_ALBEDO,
                       background=DEFAULT_BACKGROUND, step_scale: float = 0.5,
                       refine_steps: int = 8, codes: bool = False) -> torch.Tensor:
    """raycast.py:223-262: the (H, W, 3) float64 view of the isosurface on the
    device; codes=True returns quantize8's 8-bit codes (uint8) instead."""
    if step_scale <= 0.0:
        raise ValueError("step_scale must be positive")
    dev = L.require_cuda()
    shape = (cam.height, cam.width, 3)
    lo, hi = grid.value_range
    if not (lo < isovalue < hi):
        # no crossing exists anywhere, so every ray misses
        bg = torch.tensor(background, dtype=torch.float64, device=dev)
        out = bg.expand(shape).contiguous()
        if codes:
            return torch.round(torch.clamp(out, 0.0, 1.0) * 255.0).to(torch.uint8)
        return out
    data = grid.device_data(dev)
    dims, sp, org = _grid_args(grid)
    step = step_scale * float(min(grid.spacing))
    al = (ctypes.c_double * 3)(*[float(v) for v in albedo])
    bgc = (ctypes.c_double * 3)(*[float(v) for v in background])
    out = torch.empty(shape, dtype=torch.uint8 if codes else torch.float64, device=dev)
    c = L.camera_struct(cam)
    L.check(L.lib().isg_raycast(L.ptr(data), _cp(dims), _cp(sp), _cp(org), float(isovalue),
                                ctypes.byref(c), step, int(refine_steps), _cp(al), _cp(bgc),
                                None if codes else L.ptr(out), L.ptr(out) if codes else None,
                                L.stream_ptr()), "isg_raycast")
    return out


def quantize8(img) -> np.ndarray:
    """images.py:9-16: clamp to [0, 1], round to the 8-bit grid (ties to
    even), as float64."""
    q = np.rint(np.clip(np.asarray(img, dtype=np.float64), 0.0, 1.0) * 255.0)
    return q / 255.0


def gyroid_grid(n: int, periods: float) -> VolumeGrid:
    """The gyroid volume of BASELINE configs 2-4: sin x cos y +
    sin y cos z + sin z cos x at coordinate i*2*pi*periods/(n-1), spacing 1."""
    s = 2.0 * np.pi * periods / (n - 1)
    ax = np.arange(n, dtype=np.float64) * s
    sx, cx = np.sin(ax), np.cos(ax)
    data = (sx[None, None, :] * cx[None, :, None] + sx[None, :, None] * cx[:, None, None]
            + sx[:, None, None] * cx[None, None, :])
    return VolumeGrid(dims=(n, n, n), spacing=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0),
                      data=data)


def distance_field(n: int, spacing: float = 1.0) -> VolumeGrid:
    """tests/conftest.py:15-22 of the reference: distance to the lattice
    centre (the sphere of config 1)."""
    c = (n - 1) / 2.0
    ax = np.arange(n, dtype=np.float64)
    z, y, x = np.meshgrid(ax, ax, ax, indexing="ij")
    data = np.sqrt((x - c) ** 2 + (y - c) ** 2 + (z - c) ** 2) * spacing
    return VolumeGrid(dims=(n, n, n), spacing=(spacing,) * 3, origin=(0.0, 0.0, 0.0), data=data)
