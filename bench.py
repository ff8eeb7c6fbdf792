"""Benchmark: device-timed training images/s of the B200 training step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config config3]
    python bench.py --impl reference ...     # the reference's CPU path (oracle port)

Workload (BASELINE.json configs[2], the 1/2/4/8-GPU headline): Kingsnake-scale
synthetic gyroid isosurface, 4M Gaussians, 2048x2048, 448 orbit views, GT as
8-bit codes (paper_2509_05216_b200/synthetic.py).  One step = one training
iteration on one view (project, sort, bin, raster fwd, L1+D-SSIM, raster bwd,
ordered fold, chain, dense Adam over all 4M Gaussians).

Timing: W untimed warm-up steps, then K steps bracketed by a barrier and
cuda.synchronize(), CUDA events on the launching stream, max over ranks.
Every step streams the full parameter/Adam state (368 MB + 736 MB) and the
E-sized buffers, so inputs are larger than the 126 MB L2 (no flush needed).
Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "train images/s (device-timed)"
UNIT = "images/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def read_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self):
        rows = []
        for line in (self.out or "").splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[3:]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [r[0] for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or args.dist:
        import torch.distributed as dist
        # NCCL's banner / debug lines go to a file, not to the JSON stdout
        os.environ.setdefault("NCCL_DEBUG_FILE", "/tmp/isogs_nccl.%h.%p.log")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


# ----------------------------------------------------------- reference arm --

def run_reference(args, world, rank):
    """The reference's CPU path, timed on this host's cores: the oracle port
    (oracle/, bit-exact with the reference's numba kernels, tests/test_oracle_golden.py)
    running full training iterations of the same workload."""
    if rank != 0:
        return
    import numpy as np
    from oracle import oracle as O
    from oracle import train as T
    wl, cams, imgs_u8 = cpu_workload(args)
    pts = wl["points"]
    init = init_params(pts, wl["log_scales"])
    images = imgs_u8  # float32 (V, H, W, 3)
    cfg = T.Config(iterations=max(args.steps + args.warmup, 1), eval_interval=0, seed=0)
    threads = O.num_threads()
    log(f"[reference] oracle on {threads} host threads, {pts.shape[0]} Gaussians, "
        f"{images.shape[1]}^2")
    total = args.warmup + args.steps
    res = T.train_w1(images, cams, init, cfg, evaluate_views=False, max_iters=total,
                     wall_budget_s=args.cpu_budget_s)
    times = res.iter_times
    timed = times[args.warmup:] if len(times) > args.warmup else times[-1:]
    per_it = sum(timed) / len(timed)
    value = 1.0 / per_it
    wl["sample"] = (f"{len(times)} training iterations ({len(timed)} timed) of {args.config} "
                    f"({pts.shape[0]} Gaussians) at {images.shape[1]}x{images.shape[2]}; "
                    f"budget {args.cpu_budget_s:.0f}s")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_it * 1000.0,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": wl["data"], "config": wl["config"],
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": wl["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_workload(args):
    """Host copy of the workload for the CPU arm/baseline (bounded sample)."""
    import numpy as np
    import torch
    from paper_2509_05216_b200 import synthetic as S
    name = args.config
    n, periods, mp, res, nv = S.CONFIGS[name]
    res_s = args.cpu_res or res
    pos, normals = S.gyroid_points(n, periods, mp)
    ls = _host_log_scales(pos)
    cams = S.orbit(n, nv, res_s)
    # GT: target-cloud renders would need the GPU; the CPU arm trains against a
    # flat mid-grey target of the same shape (the work per step does not
    # depend on the target's content at init: it is set by the cloud).
    views = args.cpu_views
    imgs = np.full((views, res_s, res_s, 3), 0.5, dtype=np.float32)
    cams = cams[:views]
    sample = (f"{args.warmup}+{args.steps} full training iterations of {name} "
              f"({pos.shape[0]} Gaussians) at {res_s}x{res_s}")
    return ({"points": pos, "log_scales": ls, "data": "synthetic gyroid isosurface",
             "config": workload_config(name, pos.shape[0], res_s, nv),
             "sample": sample}, cams, imgs)


def _host_log_scales(points):
    """Scale seeding for the CPU arm's inputs (the reference's exact 3-NN mean
    distance, gaussians.py:124-191) on the host (scipy kd-tree), so no GPU
    kernel touches the reference arm."""
    import numpy as np
    from scipy.spatial import cKDTree
    pts = np.asarray(points, dtype=np.float64)
    d, _ = cKDTree(pts).query(pts, k=4, workers=-1)
    dist = np.maximum(np.asarray(d[:, 1:], dtype=np.float64).mean(axis=1), 1e-7)
    return np.repeat(np.log(dist)[:, None], 3, axis=1).astype(np.float32)


def workload_config(name, n, res, views):
    return {"workload": f"{name}: synthetic gyroid isosurface, {n} Gaussians, {res}x{res}, "
                        f"{views} orbit views", "gaussians": n, "resolution": res, "views": views,
            "global_batch": 1, "parallelism": "gaussian shards + pixel row bands",
            "l2": "inputs larger than L2 (params+Adam state 1.1 GB streamed per step)"}


def init_params(points, log_scales):
    import math
    import numpy as np
    n = points.shape[0]
    rot = np.zeros((n, 4), dtype=np.float32)
    rot[:, 0] = 1.0
    return {"positions": points.astype(np.float32), "log_scales": log_scales.astype(np.float32),
            "rotations": rot,
            "opacity_logits": np.full(n, math.log(0.1 / 0.9), dtype=np.float32),
            "sh_coeffs": np.zeros((n, 4, 3), dtype=np.float32)}


# ------------------------------------------------------------------ our arm --

def run_ours(args, world, rank, local):
    import numpy as np
    import torch
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200 import _lib as L
    from paper_2509_05216_b200 import synthetic as S
    from paper_2509_05216_b200.engine import PhaseTimer, Trainer
    from paper_2509_05216_b200.training import TrainConfig, build_schedule

    dev = torch.device("cuda", local if world > 1 else 0)
    if world > 1 or args.dist:
        from paper_2509_05216_b200.distributed import bench_distributed
        return bench_distributed(args, world, rank, local)
    wl = S.make_workload(args.config, dev, log=log, resolution=args.res)
    n = wl.points.shape[0]
    res = wl.resolution
    cloud = P.cloud_from_points(wl.points, wl.log_scales, 1, dev)
    iters = args.warmup + args.steps
    total = iters + (args.warm_iters + args.steps if args.warm_iters > 0 else 0)
    cfg = TrainConfig(iterations=max(total, 1), densify=False, eval_interval=0)
    scene_extent = P.TrainDataset(wl.cameras, np.zeros((len(wl.cameras), 1, 1, 3)),
                                  P.PointCloud(wl.points, wl.normals)).scene_extent
    tr = Trainer(cloud, res, res, cfg, scene_extent, dev)
    schedule = build_schedule(total, len(wl.cameras), 0)
    # warm-up
    for it in range(1, args.warmup + 1):
        v = schedule[it - 1]
        tr.step(it, wl.cameras[v], wl.images_u8[v])
    torch.cuda.synchronize()
    # ---- device-timed region
    stream = torch.cuda.current_stream()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()  # ncu --profile-from-start off sees only the timed steps
        start.record(stream)
        for it in range(args.warmup + 1, iters + 1):
            v = schedule[it - 1]
            tr.step(it, wl.cameras[v], wl.images_u8[v])
        stop.record(stream)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    ms_total = start.elapsed_time(stop)
    ms_per_step = ms_total / args.steps
    value = 1000.0 / ms_per_step
    clocks = clk.summary()
    losses = tr.loss_dev[args.warmup + 1:iters + 1].tolist()
    log(f"[ours] {ms_per_step:.3f} ms/step, {value:.1f} images/s, losses {losses[:3]}...")

    # ---- per-phase device times + pair counts for the roofline (untimed)
    timer = PhaseTimer()
    tr.r.timer = timer
    phase_steps = min(3, args.steps)
    for k in range(phase_steps):
        it = iters - phase_steps + 1 + k
        v = schedule[it - 1]
        tr.step(it, wl.cameras[v], wl.images_u8[v])
    phases = timer.phases()
    tr.r.timer = None
    phases = {k: v / phase_steps for k, v in phases.items()}
    counts = pair_counts(tr, wl, schedule[iters - 1])
    roof = roofline(phases, counts, n, args.config if args.res is None else f"{args.config}_{args.res}")
    log("[ours] phases (ms): " + ", ".join(f"{k} {v:.3f}" for k, v in phases.items()))

    # ---- end-to-end through the public API: GT H2D from pinned host + loss D2H
    e2e = end_to_end(tr, wl, schedule, args)

    # ---- second regime: the same step after more training
    warm = warm_regime(tr, wl, schedule, args) if args.warm_iters > 0 else None

    # ---- CPU baseline: the reference path (oracle port) on this host
    cpu = None if args.no_cpu_baseline else cpu_baseline(wl, args)

    # our kernels per step (CUB sort/scan passes not counted): preprocess,
    # depth_tie_fix, gather_rank, finish_counts, rank_of, emit_span,
    # tile_offsets, raster fwd, ssim_fields, ssim_adjoint, loss_finish,
    # raster bwd, ordered fold, chain (f32), Adam groups
    launches_per_step = 15
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic gyroid isosurface; GT = quantize8(raycast_isosurface) on the GPU (the reference dataset recipe, 8-bit codes)",
        "config": workload_config(args.config, n, res, len(wl.cameras)),
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
        "gpu_launches": launches_per_step * args.steps,
        "phases_ms": {k: round(v, 4) for k, v in phases.items()},
        "pairs": counts,
        "warm": warm,
    }
    print(json.dumps(line), flush=True)


def pair_counts(tr, wl, view):
    """Per-image pair counts of the forward (I_f iterated, C contributing) and
    the backward (I_b = sum of per-pixel last contributor index), counted over
    the reference's full tile lists (SURVEY 8d units; the training launches
    walk culled lists, which would shrink I_f and I_b)."""
    import torch
    r = tr.r
    r.n_contrib_out = torch.empty((r.height, r.width), dtype=torch.int32, device=r.device)
    r.n_iter_out = torch.empty((r.height, r.width), dtype=torch.int32, device=r.device)
    use = r.use_cmask
    r.use_cmask = False
    try:
        ctx = r.forward(tr.cloud, wl.cameras[view])
    finally:
        r.use_cmask = use
    out = {"M": ctx.m, "E": ctx.e, "P": r.width * r.height,
           "I_f": int(r.n_iter_out.sum(dtype=torch.int64)),
           "C": int(r.n_contrib_out.sum(dtype=torch.int64)),
           "I_b": int(r.n_last.sum(dtype=torch.int64))}
    r.n_contrib_out = r.n_iter_out = None
    return out


def roofline(phases, c, n, config="config3"):
    """Dominant kernel's achieved rate vs its roofline (SURVEY.md 8d units).

    raster fwd: 13 I_f + 9 C flops; raster bwd: 13 I_b + 55 C flops (FP32 pipe);
    byte counts for the HBM-bound stages: preprocess 92N+56M, binning 24M+24E,
    loss 36P, chain 220M, Adam 644N."""
    peaks, src = read_peaks()
    flops = {"raster_fwd": 13 * c["I_f"] + 9 * c["C"], "raster_bwd": 13 * c["I_b"] + 55 * c["C"]}
    bytes_ = {"preprocess": 92 * n + 56 * c["M"], "sort_depth": 24 * n * 8 // 3,
              "chain_adam": 644 * n + 220 * c["M"], "chain": 220 * c["M"],
              "adam": 644 * n, "loss": 36 * c["P"],
              "reduce": 36 * c["E"] + 80 * c["M"]}
    dom = max((k for k in phases if k != "host_sync"), key=lambda k: phases[k])
    ms = phases[dom]
    if dom in flops:
        fp32 = fp32_peak()
        achieved = flops[dom] / (ms * 1e-3) / 1e12
        traffic, tsrc = ncu_traffic(dom, config)
        return {"kernel": dom, "bound": "fp32", "achieved": achieved, "peak": fp32,
                "unit": "TFLOP/s", "frac": achieved / fp32 if fp32 else None,
                "traffic": traffic, "traffic_source": tsrc,
                "peak_source": "FP32 FFMA peak 148 SM x 128 lanes x 2 x max "
                "SM clock (no FP32 entry in MEASURED_PEAKS.json)",
                "algorithmic": f"{flops[dom]:.4g} flops per launch (SURVEY 8d)"}
    b = bytes_.get(dom)
    if b is None:
        return {"kernel": dom, "bound": "hbm", "achieved": None, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": None, "traffic": None}
    achieved = b / (ms * 1e-3) / 1e9
    return {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
            "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": None,
            "peak_source": src}


def ncu_traffic(kernel: str, config: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`
    from the committed ncu --set full capture (profiles/traffic_<config>.json),
    or None when no capture of this kernel/config is committed."""
    try:
        with open(os.path.join(ROOT, "profiles", f"traffic_{config}.json")) as fh:
            t = json.load(fh)[kernel]
        return t["dram_bytes_read"] + t["dram_bytes_write"], t["source"]
    except (OSError, KeyError, ValueError):
        return None, None


def fp32_peak():
    peaks, _ = read_peaks()
    mhz = peaks.get("sm_max_mhz", 1965.0)
    return 148 * 128 * 2 * mhz * 1e6 / 1e12


def end_to_end(tr, wl, schedule, args):
    """Same metric through the public Trainer.step API with each step's input
    (the view's 8-bit GT, 12.6 MB at 2K) copied H2D from pinned host memory and
    the step's loss read back D2H, all inside the timed region.  The copies are
    pipelined like a data loader would: step k+1's GT is copied on a side
    stream while step k computes (two device buffers), and step k's loss is
    read on the host (after an event sync) once step k+1 has been issued."""
    import torch
    nv = len(wl.cameras)
    host = torch.empty(wl.images_u8.shape, dtype=torch.uint8).pin_memory()
    host.copy_(wl.images_u8)
    dev = wl.images_u8.device
    gt_dev = [torch.empty(wl.images_u8.shape[1:], dtype=torch.uint8, device=dev) for _ in range(2)]
    loss_host = torch.zeros(2, dtype=torch.float64).pin_memory()
    slot = [torch.zeros(1, dtype=torch.float64, device=dev) for _ in range(2)]
    main = torch.cuda.current_stream()
    copy = torch.cuda.Stream()
    copied = [torch.cuda.Event() for _ in range(2)]
    used = [torch.cuda.Event() for _ in range(2)]
    read = [torch.cuda.Event() for _ in range(2)]
    iters = args.warmup + args.steps
    first = iters - args.steps + 1

    def prefetch(k):
        b = k % 2
        with torch.cuda.stream(copy):
            if k >= 2:
                copy.wait_event(used[b])  # step k-2 has finished reading this buffer
            gt_dev[b].copy_(host[schedule[first + k - 1]], non_blocking=True)
            copied[b].record(copy)

    losses = []
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record(main)
    prefetch(0)
    for k in range(args.steps):
        b = k % 2
        it = first + k
        main.wait_event(copied[b])
        tr.step(it, wl.cameras[schedule[it - 1]], gt_dev[b], loss_slot=slot[b])
        used[b].record(main)
        loss_host[b:b + 1].copy_(slot[b], non_blocking=True)
        read[b].record(main)
        if k + 1 < args.steps:
            prefetch(k + 1)
        if k >= 1:
            read[1 - b].synchronize()
            losses.append(float(loss_host[1 - b]))
    read[(args.steps - 1) % 2].synchronize()
    losses.append(float(loss_host[(args.steps - 1) % 2]))
    stop.record(main)
    torch.cuda.synchronize()
    ms = start.elapsed_time(stop) / args.steps
    assert len(losses) == args.steps and all(math.isfinite(x) for x in losses)
    return {"value": 1000.0 / ms, "unit": UNIT, "h2d_bytes_per_step": int(gt_dev[0].numel()),
            "d2h_bytes_per_step": 8, "ms_per_step": ms,
            "pipelining": "GT of step k+1 copied on a side stream during step k; loss of step k read after step k+1 is issued"}


def warm_regime(tr, wl, schedule, args):
    """SURVEY 8d's post-warm-up regime: args.warm_iters more (untimed)
    training iterations of the same trainer (no densification, N fixed), then
    K device-timed steps like the headline.  Opacities have grown, so pixels
    saturate and stop earlier; the pair counts say by how much."""
    import torch
    base = args.warmup + args.steps
    for it in range(base + 1, base + args.warm_iters + 1):
        v = schedule[it - 1]
        tr.step(it, wl.cameras[v], wl.images_u8[v])
    first = base + args.warm_iters + 1
    stream = torch.cuda.current_stream()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record(stream)
    for it in range(first, first + args.steps):
        v = schedule[it - 1]
        tr.step(it, wl.cameras[v], wl.images_u8[v])
    stop.record(stream)
    torch.cuda.synchronize()
    ms = start.elapsed_time(stop) / args.steps
    last = first + args.steps - 1
    loss = float(tr.loss_dev[last])
    log(f"[ours] warm regime after {first - 1} iterations: {ms:.3f} ms/step, loss {loss:.4f}")
    return {"after_iterations": first - 1, "ms_per_step": ms, "value": 1000.0 / ms,
            "unit": UNIT, "loss": loss, "pairs": pair_counts(tr, wl, schedule[last - 1])}


def cpu_baseline(wl, args):
    """The oracle port of the reference path on this host's cores: one full
    training iteration of the same workload (bounded sample)."""
    import numpy as np
    from oracle import oracle as O
    from oracle import train as T
    try:
        O.build()
        init = init_params(wl.points, wl.log_scales)
        img = wl.images_u8[:1].cpu().numpy().astype(np.float64) / 255.0
        cams = wl.cameras[:1]
        cfg = T.Config(iterations=1, eval_interval=0, seed=0)
        res = T.train_w1(img.astype(np.float32), cams, init, cfg, evaluate_views=False)
        per = res.total_wall_s
        return {"value": 1.0 / per, "unit": UNIT, "cores": O.num_threads(), "kind": "port",
                "sample": f"1 training iteration of {args.config} ({wl.points.shape[0]} "
                          f"Gaussians, {wl.resolution}^2) on the oracle (C, OpenMP)",
                "seconds": per}
    except Exception as exc:  # noqa: BLE001 -- report, never fail the bench line
        return {"value": None, "unit": UNIT, "cores": None, "kind": "port",
                "sample": f"failed: {exc!r}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="config3", choices=["config2", "config3", "config4"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--res", type=int, default=None,
                    help="override the config's image resolution (BASELINE config 5 sweep)")
    ap.add_argument("--warm-iters", type=int, default=500,
                    help="also time the post-warm-up regime after this many more "
                         "iterations (0: skip)")
    ap.add_argument("--cpu-res", type=int, default=None)
    ap.add_argument("--cpu-views", type=int, default=4)
    ap.add_argument("--cpu-budget-s", type=float, default=150.0)
    ap.add_argument("--dist", action="store_true",
                    help="run the sharded engine even at N=1 (torchrun, world 1)")
    args = ap.parse_args()
    if args.warmup < 3:
        log("[bench] warm-up raised to the required minimum of 3")
        args.warmup = 3
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        return run_reference(args, world, rank)
    world, rank, local = dist_setup(args)
    run_ours(args, world, rank, local)
    if world > 1 or args.dist:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
