"""Single-worker training loop of the reference, on the CPU oracle --
TEST INFRASTRUCTURE ONLY (tests/, smoke() checker, bench.py CPU baseline).

Follows engine._worker_run for W=1 (engine.py:465-562) with the kernels
replaced by oracle/isg_oracle.c: project -> lexsort -> tile lists -> composite
-> L1+D-SSIM -> per-tile backward -> ascending-tile fold -> stats -> chain ->
dense Adam.  Densification is not restated (it never triggers in the configs
this loop is used for: densify_start=500 > iterations/2).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import oracle as O

PARAM_NAMES = ("positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs")


def build_schedule(iterations: int, n_views: int, seed: int) -> list[int]:
    """engine.py:602-610."""
    out: list[int] = []
    epoch = 0
    while len(out) < iterations:
        rng = np.random.default_rng((int(seed), int(epoch)))
        out.extend(int(v) for v in rng.permutation(n_views))
        epoch += 1
    return out[:iterations]


def position_lr(base_lr: float, iteration: int, total: int, final_mult: float = 0.01) -> float:
    """optim.py:59-64."""
    if total <= 0:
        return base_lr
    t = min(max(iteration, 0), total) / total
    return base_lr * (final_mult ** t)


def scene_extent(cameras) -> float:
    """training.py:262-267."""
    pos = np.stack([-np.asarray(c.rotation).T @ np.asarray(c.translation) for c in cameras])
    centroid = pos.mean(axis=0)
    ext = float(np.linalg.norm(pos - centroid, axis=1).max())
    return ext if ext > 0 else 1.0


@dataclass
class Config:
    """The TrainConfig fields the hot path reads (training.py:34-56)."""

    iterations: int = 2000
    lambda_dssim: float = 0.2
    lr_position: float = 1.6e-4
    lr_position_final: float = 0.01
    lr_sh: float = 2.5e-3
    lr_opacity: float = 5e-2
    lr_scale: float = 5e-3
    lr_rotation: float = 1e-3
    seed: int = 0
    background: tuple = (1.0, 1.0, 1.0)
    eval_interval: int = 0
    sh_degree: int = 1
    tile_size: int = 16


@dataclass
class Record:
    iteration: int
    loss: float
    psnr: float
    ssim: float


@dataclass
class Result:
    params: dict
    losses: list = field(default_factory=list)
    records: list = field(default_factory=list)
    total_wall_s: float = 0.0


class _CloudView:
    def __init__(self, params, degree):
        self.positions = params["positions"]
        self.log_scales = params["log_scales"]
        self.rotations = params["rotations"]
        self.opacity_logits = params["opacity_logits"]
        self.sh_coeffs = params["sh_coeffs"]
        self.degree = degree


def render_view(params, degree, cam, cfg: Config):
    """engine.py:184-253 for W=1: returns (canvas f32, context)."""
    cloud = _CloudView(params, degree)
    batch = O.project(cloud, cam, cfg.tile_size)
    img, aux, order = O.render_forward(batch, cam.width, cam.height, cfg.background,
                                       cfg.tile_size, dtype=np.float32)
    return img, (cloud, batch, aux, order)


def evaluate(params, degree, cameras, images, cfg: Config, it: int) -> Record:
    """engine.py:440-462 + training.py:392-396."""
    losses, psnrs, ssims = [], [], []
    for v, cam in enumerate(cameras):
        img, _ = render_view(params, degree, cam, cfg)
        ref = images[v]
        losses.append(O.loss_l1_dssim(img, ref, cfg.lambda_dssim)[0])
        a = O.quantize8(img)
        b = O.quantize8(ref)
        psnrs.append(O.psnr(a, b))
        ssims.append(O.ssim(a, b))
    return Record(it, float(np.mean(losses)), float(np.mean(psnrs)), float(np.mean(ssims)))


def iteration(params: dict, state: dict, seen, grad_accum, degree: int, it: int, cam, ref,
              cfg: Config, extent: float):
    """One W=1 training iteration in place (engine.py:481-537): render, loss,
    backward, 2-D fold, stats, chain, Adam.  Returns (loss, details) with the
    iteration's canvas, parameter gradients, 2-D gradients (cloud row order)
    and visible rows."""
    n = params["positions"].shape[0]
    h, w = ref.shape[0], ref.shape[1]
    img, (cloud, batch, aux, order) = render_view(params, degree, cam, cfg)
    loss, dimg = O.loss_l1_dssim(img, ref, cfg.lambda_dssim)
    b2d, _ = O.render_backward_2d(batch, order, aux, dimg)
    rows = batch.indices
    full = {k: np.zeros((n,) + v.shape[1:]) for k, v in b2d.items()}
    for k in full:
        full[k][rows] = b2d[k]
    seen[rows] += 1
    grad_accum[rows] += np.hypot(full["dmean"][rows, 0] * (0.5 * w),
                                 full["dmean"][rows, 1] * (0.5 * h))
    flags = np.zeros(n, dtype=np.uint8)
    flags[rows] = 1
    pg = O.chain_to_params(cloud, cam, flags, full["dmean"], full["dconic"],
                           full["dcolor"], full["dopac"])
    grads = {k: getattr(pg, k) for k in PARAM_NAMES}
    lrs = {
        "positions": extent * position_lr(cfg.lr_position, it, cfg.iterations,
                                          cfg.lr_position_final),
        "log_scales": cfg.lr_scale,
        "rotations": cfg.lr_rotation,
        "opacity_logits": cfg.lr_opacity,
        "sh_coeffs": cfg.lr_sh,
    }
    details = {"iteration": it, "image": img, "loss": float(loss),
               "param_grads": {k: np.array(v, copy=True) for k, v in grads.items()},
               "grad2d": full, "visible": rows.copy(), "lrs": lrs,
               "depth_order_rows": rows[order].copy(), "offsets": aux.cache["offsets"],
               "entries": aux.cache["entries"]}
    O.adam_step(params, grads, state, it, lrs)
    return float(loss), details


def train_w1(images, cameras, init_params: dict, cfg: Config, extent: float | None = None,
             evaluate_views: bool = True, max_iters: int | None = None,
             wall_budget_s: float | None = None, schedule=None,
             keep_grads: bool = False) -> Result:
    """engine.py:465-562 with W=1.  ``max_iters`` / ``wall_budget_s`` stop early
    (the schedule and learning rates still follow cfg.iterations), used for
    bounded CPU samples; per-iteration wall times land in Result.iter_times.
    ``schedule`` overrides the view order (indices into ``cameras``);
    ``keep_grads`` keeps the last iteration's parameter gradients, 2-D
    gradients (cloud row order) and canvas in Result.last."""
    params = {k: np.array(init_params[k], dtype=np.float32, copy=True) for k in PARAM_NAMES}
    state = {k: {"m": np.zeros_like(v), "v": np.zeros_like(v)} for k, v in params.items()}
    degree = cfg.sh_degree
    n = params["positions"].shape[0]
    seen = np.zeros(n, dtype=np.int64)
    grad_accum = np.zeros(n, dtype=np.float64)
    if extent is None:
        extent = scene_extent(cameras)
    h, w = images.shape[1], images.shape[2]
    res = Result(params=params)
    res.iter_times = []
    if evaluate_views:
        res.records.append(evaluate(params, degree, cameras, images, cfg, 0))
    if schedule is None:
        schedule = build_schedule(cfg.iterations, len(cameras), cfg.seed)
    last = cfg.iterations if max_iters is None else min(max_iters, cfg.iterations)
    for it in range(1, last + 1):
        t0 = time.perf_counter()
        cam = cameras[schedule[it - 1]]
        ref = images[schedule[it - 1]]
        loss, det = iteration(params, state, seen, grad_accum, degree, it, cam, ref, cfg, extent)
        if keep_grads:
            res.last = det
        dt = time.perf_counter() - t0
        res.total_wall_s += dt
        res.iter_times.append(dt)
        res.losses.append(float(loss))
        due = it == cfg.iterations or (cfg.eval_interval > 0 and it % cfg.eval_interval == 0)
        if evaluate_views and due:
            res.records.append(evaluate(params, degree, cameras, images, cfg, it))
        if wall_budget_s is not None and res.total_wall_s >= wall_budget_s:
            break
    res.seen = seen
    res.grad_accum = grad_accum
    return res
