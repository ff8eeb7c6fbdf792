"""Clone / split / prune by accumulated gradient statistics, on the device.

Mirrors the reference's densify_and_prune (src/isosplat/training.py:315-389)
and the single-worker bookkeeping of _densify_step (src/isosplat/engine.py:
307-382): rows are classified from TrainStats and the activated scales and
opacities, survivors are re-ordered as kept rows (ascending), clones (by
parent), then the two children of every split parent; kept rows carry their
Adam moments, new rows start cold, and the statistics restart at zero.

The reference classifies with numpy (np.exp of the log-scales and logits,
float64); here the classification runs on the device in float64 with the
glibc-exact exp (isg_densify_classify, the same bits), and only the split
parents' rows go to the host.  Split children are drawn exactly as the reference draws them:
one numpy Generator per parent seeded by (seed, iteration, global id), for
the split rows only.  Densify runs every densify_interval steps; it is not
on the per-iteration path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from .gaussians import PARAM_NAMES, GaussianCloud
from .training import TrainStats

SPLIT_SCALE_SHRINK = 1.6  # training.py:20
SPLIT_EXTENT_FRACTION = 0.01  # training.py:21


@dataclass
class DensifyMapping:
    """Row bookkeeping of one densify/prune event (training.py:300-312);
    int64 row indices into the cloud before the event."""

    kept: torch.Tensor
    cloned: torch.Tensor
    split: torch.Tensor
    pruned: torch.Tensor

    @property
    def identity(self) -> bool:
        return self.cloned.numel() == 0 and self.split.numel() == 0 and self.pruned.numel() == 0


def _quat_to_rotation(q: np.ndarray) -> np.ndarray:
    """gaussians.quat_to_rotation (gaussians.py:81-92), float64, one row."""
    n = np.linalg.norm(q)
    if n < 1e-12:
        raise ValueError("zero-norm quaternion")
    w, x, y, z = q / n
    return np.array([
        [1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y)],
        [2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x)],
        [2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)],
    ])


def classify(log_scales: np.ndarray, opacity_logits: np.ndarray, seen: np.ndarray,
             grad_accum: np.ndarray, opacity_prune: float, scale_prune: float,
             grad_threshold: float, split_threshold: float):
    """prune / split / clone / keep masks and the float64 activated scales,
    statement for statement as training.py:334-347 (host numpy arrays)."""
    avg = grad_accum / np.maximum(seen, 1)
    scales = np.exp(log_scales.astype(np.float64))
    max_scale = scales.max(axis=1)
    opacity = 1.0 / (1.0 + np.exp(-opacity_logits.astype(np.float64)))
    prune = opacity < opacity_prune
    if np.isfinite(scale_prune):
        prune |= max_scale > scale_prune
    hot = (avg > grad_threshold) & ~prune
    split = hot & (max_scale > split_threshold)
    clone = hot & ~split
    keep = ~(prune | split)
    return keep, clone, split, prune, scales


def densify_and_prune(cloud: GaussianCloud, stats: TrainStats, config, iteration: int,
                      grad_threshold: float, split_threshold: float,
                      global_ids=None) -> tuple[GaussianCloud, DensifyMapping]:
    """training.py:315-389 on the device.  New row order: kept, clones,
    then the children of every split parent (two each, parent order)."""
    n = cloud.count
    dev = cloud.positions.device
    if global_ids is None:
        gids = np.arange(n, dtype=np.int64)
    else:
        gids = np.asarray(global_ids.cpu() if isinstance(global_ids, torch.Tensor)
                          else global_ids, dtype=np.int64)
        if gids.shape != (n,):
            raise ValueError("global_ids must have one id per row")
    if dev.type == "cuda" and cloud.positions.dtype == torch.float32:
        # classification on the device (isg_densify_classify: float64, the
        # glibc-exact exp); only the split parents' rows come to the host
        cls = _classify_device(cloud, stats, config, grad_threshold, split_threshold)
        kept_rows = torch.nonzero(cls <= 1).flatten()
        clone_rows = torch.nonzero(cls == 1).flatten()
        split_rows = torch.nonzero(cls == 2).flatten()
        prune_rows = torch.nonzero(cls == 3).flatten()
        rows_h = split_rows.cpu().numpy()
        scales = None
    else:  # host tensors (the gloo tests of the sharded bookkeeping)
        keep, clone, split, prune, scales = classify(
            cloud.log_scales.cpu().numpy(), cloud.opacity_logits.cpu().numpy(),
            _host(stats.seen, np.int64), _host(stats.grad_accum, np.float64),
            config.opacity_prune, config.scale_prune, grad_threshold, split_threshold)
        rows = {}
        for name, mask in (("kept", keep), ("clone", clone), ("split", split),
                           ("prune", prune)):
            rows[name] = torch.from_numpy(np.nonzero(mask)[0].astype(np.int64)).to(dev)
        kept_rows, clone_rows, split_rows, prune_rows = (rows["kept"], rows["clone"],
                                                         rows["split"], rows["prune"])
        rows_h = np.nonzero(split)[0]
    parts = {k: [getattr(cloud, k)[kept_rows], getattr(cloud, k)[clone_rows]]
             for k in PARAM_NAMES}
    ns = int(split_rows.numel())
    if ns:
        dt = cloud.positions.dtype
        sc_h = (scales[rows_h] if scales is not None else
                np.exp(cloud.log_scales[split_rows].cpu().numpy().astype(np.float64)))
        rot_h = cloud.rotations[split_rows].cpu().numpy().astype(np.float64)
        pos_h = cloud.positions[split_rows].cpu().numpy().astype(np.float64)
        child = np.empty((2 * ns, 3), dtype=np.float64)
        seed = int(config.seed)
        for j in range(ns):
            rng = np.random.default_rng((seed, int(iteration), int(gids[rows_h[j]])))
            offs = rng.standard_normal((2, 3)) * sc_h[j]
            rot = _quat_to_rotation(rot_h[j])
            child[2 * j] = pos_h[j] + rot @ offs[0]
            child[2 * j + 1] = pos_h[j] + rot @ offs[1]
        rep = torch.repeat_interleave(split_rows, 2)
        np_dt = np.float32 if dt == torch.float32 else np.float64
        parts["positions"].append(torch.from_numpy(child.astype(np_dt)).to(dev))
        parts["log_scales"].append(
            (cloud.log_scales[rep].to(torch.float64) - math.log(SPLIT_SCALE_SHRINK)).to(dt))
        for k in ("rotations", "opacity_logits", "sh_coeffs"):
            parts[k].append(getattr(cloud, k)[rep])
    new = GaussianCloud(*(torch.cat(parts[k]).contiguous() for k in PARAM_NAMES),
                        degree=cloud.degree)
    return new, DensifyMapping(kept=kept_rows, cloned=clone_rows, split=split_rows,
                               pruned=prune_rows)


def _classify_device(cloud: GaussianCloud, stats: TrainStats, config, grad_threshold: float,
                     split_threshold: float) -> torch.Tensor:
    """Per-row class (0 keep, 1 clone, 2 split, 3 prune) by isg_densify_classify."""
    import ctypes
    from . import _lib as L
    n = cloud.count
    cls = torch.empty(n, dtype=torch.uint8, device=cloud.positions.device)
    seen = stats.seen.to(device=cls.device, dtype=torch.int64).contiguous()
    acc = stats.grad_accum.to(device=cls.device, dtype=torch.float64).contiguous()
    sp = float(config.scale_prune)
    on = 1 if math.isfinite(sp) else 0
    L.check(L.lib().isg_densify_classify(
        n, L.ptr(cloud.log_scales), L.ptr(cloud.opacity_logits), L.ptr(seen), L.ptr(acc),
        float(config.opacity_prune), sp if on else 0.0, on, float(grad_threshold),
        float(split_threshold), L.ptr(cls), L.stream_ptr()), "isg_densify_classify")
    return cls


def _host(x, dtype) -> np.ndarray:
    a = x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)
    return a.astype(dtype, copy=False)


def carry_moments(state: dict, mapping: DensifyMapping, new: GaussianCloud) -> dict:
    """Kept rows keep their Adam moments, clones and children start at zero
    (engine.py:374-381)."""
    out = {}
    kn = int(mapping.kept.numel())
    for k in PARAM_NAMES:
        fresh = torch.zeros_like(getattr(new, k))
        if kn:
            fresh[:kn] = state[k][mapping.kept]
        out[k] = fresh
    return out
