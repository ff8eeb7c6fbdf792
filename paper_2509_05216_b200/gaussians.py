"""Gaussian parameter storage on the device (reference gaussians.py:27-78).

Parameters are pre-activation and keep the reference's row-major layout per
parameter -- positions (N,3), log_scales (N,3), rotations (N,4) wxyz,
opacity_logits (N,), sh_coeffs (N,K,3) -- as CUDA tensors, float32 for
training (float64 accepted by the API for the tight cross-check build).
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass

import numpy as np
import torch

PARAM_NAMES = ("positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs")
_INIT_OPACITY_LOGIT = math.log(0.1 / 0.9)
_CKPT_MAGIC = b"SSGC"  # gaussians.py:18-19
_CKPT_VERSION = 1


@dataclass
class GaussianCloud:
    positions: torch.Tensor
    log_scales: torch.Tensor
    rotations: torch.Tensor
    opacity_logits: torch.Tensor
    sh_coeffs: torch.Tensor
    degree: int = 1

    @property
    def count(self) -> int:
        return int(self.positions.shape[0])

    @property
    def dtype(self) -> torch.dtype:
        return self.positions.dtype

    def validate(self) -> None:
        n = self.count
        k = (self.degree + 1) ** 2
        if self.degree not in (0, 1):
            raise ValueError(f"degree must be 0 or 1, got {self.degree}")
        want = {"positions": (n, 3), "log_scales": (n, 3), "rotations": (n, 4),
                "opacity_logits": (n,), "sh_coeffs": (n, k, 3)}
        for name, shape in want.items():
            got = tuple(getattr(self, name).shape)
            if got != shape:
                raise ValueError(f"{name}: shape {got}, expected {shape}")

    def copy(self) -> "GaussianCloud":
        return GaussianCloud(*(getattr(self, k).clone() for k in PARAM_NAMES), degree=self.degree)

    def numpy(self) -> dict:
        return {k: getattr(self, k).detach().cpu().numpy() for k in PARAM_NAMES}


def to_device_cloud(cloud, device=None, dtype: torch.dtype | None = None) -> GaussianCloud:
    """Any object with the reference's cloud attributes (numpy or torch) ->
    contiguous CUDA GaussianCloud (dtype preserved unless given)."""
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())

    def conv(a):
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
        if dtype is not None:
            t = t.to(dtype)
        elif t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float32)
        return t.to(device).contiguous()

    out = GaussianCloud(*(conv(getattr(cloud, k)) for k in PARAM_NAMES),
                        degree=int(cloud.degree))
    dt = out.positions.dtype
    for k in PARAM_NAMES:
        if getattr(out, k).dtype != dt:
            setattr(out, k, getattr(out, k).to(dt))
    return out


def cloud_from_points(points: np.ndarray, log_scales: np.ndarray, degree: int = 1,
                      device=None) -> GaussianCloud:
    """init_from_points (gaussians.py:165-191) with precomputed log-scales:
    identity rotation, opacity 0.1, zero SH."""
    n = points.shape[0]
    k = (degree + 1) ** 2
    rot = np.zeros((n, 4), dtype=np.float32)
    rot[:, 0] = 1.0
    ls = np.asarray(log_scales, dtype=np.float32)
    if ls.ndim == 1:
        ls = np.repeat(ls[:, None], 3, axis=1)
    host = GaussianCloud(
        positions=torch.from_numpy(np.asarray(points, dtype=np.float32)),
        log_scales=torch.from_numpy(np.ascontiguousarray(ls)),
        rotations=torch.from_numpy(rot),
        opacity_logits=torch.from_numpy(np.full(n, _INIT_OPACITY_LOGIT, dtype=np.float32)),
        sh_coeffs=torch.from_numpy(np.zeros((n, k, 3), dtype=np.float32)),
        degree=degree)
    return to_device_cloud(host, device)


def save_checkpoint(path: str, cloud) -> None:
    """The reference's SSGC file (gaussians.py:194-204): magic, <IQI version /
    count / degree, then the five parameter blocks as little-endian float32.
    Accepts a device GaussianCloud or any object with the cloud attributes."""
    n = int(cloud.positions.shape[0])
    deg = int(cloud.degree)
    with open(path, "wb") as fh:
        fh.write(_CKPT_MAGIC)
        fh.write(struct.pack("<IQI", _CKPT_VERSION, n, deg))
        for k in PARAM_NAMES:
            a = getattr(cloud, k)
            a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
            fh.write(np.ascontiguousarray(a, dtype="<f4").tobytes())


def load_checkpoint(path: str, device=None) -> GaussianCloud:
    """Read an SSGC file (gaussians.py:206-235, same validation errors) into
    a float32 device cloud."""
    with open(path, "rb") as fh:
        blob = fh.read()
    if blob[:4] != _CKPT_MAGIC:
        raise ValueError(f"{path}: bad magic {blob[:4]!r}, expected {_CKPT_MAGIC!r}")
    version, n, degree = struct.unpack_from("<IQI", blob, 4)
    if version != _CKPT_VERSION:
        raise ValueError(f"{path}: unsupported version {version}")
    k = (degree + 1) ** 2
    counts = [n * 3, n * 3, n * 4, n, n * k * 3]
    body = 4 + struct.calcsize("<IQI")
    want = body + 4 * sum(counts)
    if len(blob) != want:
        raise ValueError(f"{path}: expected {want} bytes, got {len(blob)}")
    flat = np.frombuffer(blob, dtype="<f4", offset=body)
    shapes = [(n, 3), (n, 3), (n, 4), (n,), (n, k, 3)]
    parts, at = [], 0
    for c, shp in zip(counts, shapes):
        parts.append(flat[at:at + c].reshape(shp).astype(np.float32))
        at += c
    host = GaussianCloud(*(torch.from_numpy(p_) for p_ in parts), degree=int(degree))
    host.validate()
    return to_device_cloud(host, device)


def save_train_state(path: str, trainer, iteration: int) -> None:
    """Resumable training state (an extension: the reference checkpoint holds
    parameters only): the SSGC cloud plus Adam moments, TrainStats and the
    iteration in `path + '.state.npz'`."""
    save_checkpoint(path, trainer.cloud)
    extra = {"iteration": np.array(iteration)}
    for k in PARAM_NAMES:
        extra["m_" + k] = trainer.m[k].cpu().numpy()
        extra["v_" + k] = trainer.v[k].cpu().numpy()
    extra["seen"] = trainer.stats.seen.cpu().numpy()
    extra["grad_accum"] = trainer.stats.grad_accum.cpu().numpy()
    np.savez(path + ".state.npz", **extra)


def load_train_state(path: str, trainer) -> int:
    """Restore a Trainer from save_train_state; returns the iteration."""
    from .training import TrainStats
    cloud = load_checkpoint(path, trainer.device)
    z = np.load(path + ".state.npz")
    dev = trainer.device
    trainer.cloud = cloud
    trainer.m = {k: torch.from_numpy(z["m_" + k]).to(dev) for k in PARAM_NAMES}
    trainer.v = {k: torch.from_numpy(z["v_" + k]).to(dev) for k in PARAM_NAMES}
    trainer.stats = TrainStats(grad_accum=torch.from_numpy(z["grad_accum"]).to(dev),
                               seen=torch.from_numpy(z["seen"]).to(dev))
    trainer.grads = None
    return int(z["iteration"])
