"""Training configuration, dataset and report types (reference training.py).

The hot-path fields and semantics of TrainConfig, TrainDataset, TrainStats,
EvalRecord and TrainReport are kept verbatim so a reference user can switch.
Densification (training.py:315-389) lives in densify.py.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

BASE_RESOLUTION = 512.0


@dataclass
class TrainConfig:
    """Hyperparameters and run controls (training.py:24-121)."""

    iterations: int = 2000
    lambda_dssim: float = 0.2
    lr_position: float = 1.6e-4
    lr_position_final: float = 0.01
    lr_sh: float = 2.5e-3
    lr_opacity: float = 5e-2
    lr_scale: float = 5e-3
    lr_rotation: float = 1e-3
    densify: bool = True
    densify_interval: int = 100
    densify_start: int = 500
    densify_stop: int | None = None
    grad_threshold: float = 2e-4
    opacity_prune: float = 0.005
    scale_prune: float = math.inf
    split_threshold: float | None = None
    rebalance: bool = True
    seed: int = 0
    resolution: int | None = None
    background: tuple = (1.0, 1.0, 1.0)
    eval_interval: int = 0
    sh_degree: int = 1
    tile_size: int = 16

    def validate(self) -> None:
        if self.iterations < 0:
            raise ValueError("iterations must be >= 0")
        if not 0.0 <= self.lambda_dssim <= 1.0:
            raise ValueError("lambda_dssim must lie in [0, 1]")
        for name in ("grad_threshold", "opacity_prune", "scale_prune"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be >= 0")
        for name in ("lr_position", "lr_sh", "lr_opacity", "lr_scale", "lr_rotation"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")
        if self.densify_interval < 1:
            raise ValueError("densify_interval must be >= 1")
        if self.tile_size < 1:
            raise ValueError("tile_size must be >= 1")
        if self.sh_degree not in (0, 1):
            raise ValueError("sh_degree must be 0 or 1")
        if self.eval_interval < 0:
            raise ValueError("eval_interval must be >= 0")

    def effective_densify_stop(self) -> int:
        return self.iterations // 2 if self.densify_stop is None else self.densify_stop

    def effective_grad_threshold(self, resolution: int) -> float:
        return self.grad_threshold * (resolution / BASE_RESOLUTION)

    def densify_active(self) -> bool:
        """True if the schedule would run densify_and_prune at least once
        (engine.py:540-541)."""
        if not self.densify:
            return False
        stop = self.effective_densify_stop()
        first = max(self.densify_start, self.densify_interval)
        first = ((first + self.densify_interval - 1) // self.densify_interval) * self.densify_interval
        return first <= min(stop, self.iterations)


@dataclass
class PointCloud:
    """volume.py PointCloud: positions and normals (N, 3)."""

    positions: np.ndarray
    normals: np.ndarray

    @property
    def count(self) -> int:
        return int(self.positions.shape[0])


@dataclass
class EvalRecord:
    iteration: int
    loss: float
    psnr: float
    ssim: float
    wall_s: float
    gaussians: int


@dataclass
class TrainReport:
    """training.py:159-219 (records, losses, wall, phase rows)."""

    workers: int
    resolution: int
    records: list = field(default_factory=list)
    iteration_losses: list = field(default_factory=list)
    total_wall_s: float = 0.0
    phase_rows: list = field(default_factory=list)

    @property
    def final(self) -> EvalRecord:
        return self.records[-1]


def deterministic_equal(a: TrainReport, b: TrainReport) -> bool:
    """training.py:222-233."""
    if a.workers != b.workers or a.resolution != b.resolution:
        return False
    if len(a.records) != len(b.records):
        return False
    for ra, rb in zip(a.records, b.records):
        if (ra.iteration, ra.gaussians, ra.loss, ra.psnr, ra.ssim) != \
                (rb.iteration, rb.gaussians, rb.loss, rb.psnr, rb.ssim):
            return False
    return a.iteration_losses == b.iteration_losses


@dataclass
class TrainDataset:
    """Reference views plus the seeding point cloud (training.py:236-267).

    images: (V, H, W, 3) float32 in [0, 1] (or uint8 8-bit codes)."""

    cameras: list
    images: np.ndarray
    points: PointCloud

    def __post_init__(self) -> None:
        if len(self.cameras) == 0:
            raise ValueError("dataset has no views")
        if self.images.shape[0] != len(self.cameras):
            raise ValueError("one image per camera required")

    @property
    def view_count(self) -> int:
        return len(self.cameras)

    @property
    def width(self) -> int:
        return int(self.images.shape[2])

    @property
    def height(self) -> int:
        return int(self.images.shape[1])

    @property
    def scene_extent(self) -> float:
        pos = np.stack([c.position for c in self.cameras])
        centroid = pos.mean(axis=0)
        ext = float(np.linalg.norm(pos - centroid, axis=1).max())
        return ext if ext > 0 else 1.0


@dataclass
class TrainStats:
    """Densification accumulators (training.py:287-297), on the device."""

    grad_accum: object
    seen: object


def build_schedule(iterations: int, n_views: int, seed: int) -> list[int]:
    """Deterministic epoch shuffle (engine.py:602-610)."""
    out: list[int] = []
    epoch = 0
    while len(out) < iterations:
        rng = np.random.default_rng((int(seed), int(epoch)))
        out.extend(int(v) for v in rng.permutation(n_views))
        epoch += 1
    return out[:iterations]


def mean_knn_distance(points: np.ndarray, k: int = 3) -> np.ndarray:
    """Mean distance to the k nearest neighbours (gaussians.py:124-162) on the
    GPU (isg_knn_mean_grid): the bucket grid is set up on the host exactly as
    the reference does it with numpy, the ring search runs one thread per
    point.  Bit-exact with the reference's grid path (n > 10000); for smaller
    clouds the reference uses a brute-force partition whose summation order is
    unspecified (last-bit differences possible)."""
    import ctypes
    import torch
    from . import _lib as L
    pts = np.ascontiguousarray(points, dtype=np.float64)
    n = pts.shape[0]
    kk = min(k, n - 1)
    if kk <= 0:
        return np.ones(n)
    lo = pts.min(axis=0)
    hi = pts.max(axis=0)
    span = np.maximum(hi - lo, 1e-12)
    cell = float(np.cbrt(span.prod() / n)) * 2.0
    if cell <= 0.0 or not np.isfinite(cell):
        cell = float(span.max()) or 1.0
    dims = (np.floor((hi - lo) / cell)).astype(np.int64) + 1
    dev = L.require_cuda()
    d_pts = torch.from_numpy(pts).to(dev)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    lo_c = (ctypes.c_double * 3)(*lo.tolist())
    sz = ctypes.c_size_t(0)
    lib = L.lib()
    args = (n, kk, ctypes.cast(lo_c, ctypes.c_void_p), cell, int(dims[0]), int(dims[1]),
            int(dims[2]))
    L.check(lib.isg_knn_mean_grid(None, ctypes.byref(sz), None, *args, None, None),
            "isg_knn_mean_grid (size)")
    ws = torch.empty(max(sz.value, 1), dtype=torch.uint8, device=dev)
    sz = ctypes.c_size_t(ws.numel())
    L.check(lib.isg_knn_mean_grid(L.ptr(ws), ctypes.byref(sz), L.ptr(d_pts), *args, L.ptr(out),
                                  L.stream_ptr()), "isg_knn_mean_grid")
    return out.cpu().numpy()


def init_log_scales(points: np.ndarray) -> np.ndarray:
    """gaussians.py:165-191: isotropic log(mean 3-NN distance), floored at 1e-7."""
    dist = np.maximum(mean_knn_distance(np.asarray(points, dtype=np.float64)), 1e-7)
    return np.repeat(np.log(dist)[:, None], 3, axis=1).astype(np.float32)
