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


# The JSON line is the only thing on stdout: emit() writes it to a private
# duplicate of fd 1 while fd 1 itself is pointed at stderr, so library output
# (NCCL's banner and INFO lines, CUDA/C prints) cannot interleave with it.
_JSON_OUT = None


def _claim_stdout():
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)
    return _JSON_OUT


def emit(line: dict) -> None:
    out = _claim_stdout()
    out.write(json.dumps(line) + "\n")
    out.flush()


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
        # NCCL's communicator lines (rank count, transports) go to fd 1, which
        # _claim_stdout() has pointed at stderr
        if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION", "WARN"):
            os.environ["NCCL_DEBUG"] = "INFO"
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


# ----------------------------------------------------------- reference arm --

def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def total_iterations(args) -> int:
    """TrainConfig.iterations of a bench run (the position-lr schedule and the
    view schedule follow it); the same for both arms."""
    iters = args.warmup + args.steps
    return max(iters + (args.warm_iters + args.steps if args.warm_iters > 0 else 0), 1)


def host_state(points, log_scales):
    """Initial parameters (init_from_points, gaussians.py:165-191) and zero
    Adam moments / stats as host arrays for the oracle."""
    import numpy as np
    init = init_params(points, log_scales)
    n = init["positions"].shape[0]
    state = {k: {"m": np.zeros_like(v), "v": np.zeros_like(v)} for k, v in init.items()}
    return init, state, np.zeros(n, dtype=np.int64), np.zeros(n, dtype=np.float64)


def run_reference(args, world, rank):
    """The reference's CPU path, timed on this host's cores: the oracle port
    (oracle/, bit-exact with the reference's numba kernels,
    tests/test_oracle_golden.py) running full training iterations of the same
    workload -- the same points, scale init, orbit views and raycast GT codes
    as our arm (the dataset is generated before timing; on a GPU box with the
    GPU generator, bit-exact with the reference's, else on the host) -- one
    iteration per step, as many steps as fit in --cpu-budget-s."""
    if rank != 0:
        return
    import numpy as np
    from oracle import oracle as O
    from oracle import train as T
    O.build()
    wl = reference_workload(args)
    threads = O.num_threads()
    total = total_iterations(args)
    cfg = T.Config(iterations=total, eval_interval=0, seed=0)
    params, state, seen, gacc = host_state(wl["points"], wl["log_scales"])
    log(f"[reference] oracle on {threads} host threads ({cpu_model()}), "
        f"{wl['points'].shape[0]} Gaussians, {wl['res']}^2")
    # no JIT to warm: one untimed iteration pays the first-touch page faults
    warm = 1
    times = []
    for it in range(1, warm + args.steps + 1):
        k = it - 1
        t0 = time.perf_counter()
        T.iteration(params, state, seen, gacc, 1, it, wl["cameras"][k], wl["images"][k], cfg,
                    wl["extent"])
        dt = time.perf_counter() - t0
        if it > warm:
            times.append(dt)
        log(f"[reference] iteration {it}: {dt:.2f}s")
        if sum(times) >= args.cpu_budget_s:
            break
    per_it = sum(times) / len(times)
    value = 1.0 / per_it
    sample = (f"{len(times)} timed training iterations (+{warm} untimed) of {args.config} "
              f"({wl['points'].shape[0]} Gaussians, {wl['res']}x{wl['res']}, the schedule's views "
              f"and raycast GT), stopped at a {args.cpu_budget_s:.0f}s budget of the "
              f"{args.steps} requested")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": len(times), "warmup": warm, "ms_per_step": per_it * 1000.0,
        "requested": {"steps": args.steps, "warmup": args.warmup},
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": wl["data"], "config": wl["config"],
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample, "cpu_model": cpu_model(),
                         "host_cpus": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


def reference_workload(args):
    """Host copy of the workload for the reference arm: the views the first
    (1 + steps) iterations of the schedule visit, with their GT codes."""
    import numpy as np
    import torch
    from paper_2509_05216_b200 import synthetic as S
    from paper_2509_05216_b200.training import TrainDataset, PointCloud, build_schedule
    name = args.config
    n, periods, mp, res, nv = S.CONFIGS[name]
    res = args.res or res
    sched = build_schedule(total_iterations(args), nv, 0)[:args.steps + 1]
    if torch.cuda.is_available():
        wl = S.make_workload(name, torch.device("cuda", 0), view_ids=sched, resolution=res,
                             log=log)
        pos, normals, ls, cams = wl.points, wl.normals, wl.log_scales, wl.cameras
        codes = wl.images_u8.cpu().numpy()
        del wl
        torch.cuda.empty_cache()
        data = ("synthetic gyroid isosurface; GT = quantize8(raycast_isosurface), the reference "
                "dataset recipe, generated before timing")
    else:  # no GPU: host points + kNN, flat target (the work per step is set by the cloud)
        pos, normals = S.gyroid_points(n, periods, mp)
        ls = _host_log_scales(pos)
        cams = S.orbit(n, nv, res)
        codes = np.full((len(sched), res, res, 3), 128, dtype=np.uint8)
        data = "synthetic gyroid isosurface; flat GT (no GPU for the dataset generator)"
    ext = TrainDataset(cams, np.zeros((nv, 1, 1, 3)), PointCloud(pos, normals)).scene_extent
    images = (codes.astype(np.float64) / 255.0).astype(np.float32)
    return {"points": pos, "log_scales": ls, "cameras": [cams[v] for v in sched],
            "images": images, "extent": ext, "res": res, "data": data,
            "config": workload_config(name, pos.shape[0], res, nv)}


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

    dev = torch.device("cuda", 0)
    wl = S.make_workload(args.config, dev, log=log, resolution=args.res)
    n = wl.points.shape[0]
    res = wl.resolution
    cloud = P.cloud_from_points(wl.points, wl.log_scales, 1, dev)
    iters = args.warmup + args.steps
    total = total_iterations(args)
    cfg = TrainConfig(iterations=total, densify=False, eval_interval=0)
    scene_extent = P.TrainDataset(wl.cameras, np.zeros((len(wl.cameras), 1, 1, 3)),
                                  P.PointCloud(wl.points, wl.normals)).scene_extent
    tr = Trainer(cloud, res, res, cfg, scene_extent, dev)
    schedule = build_schedule(total, len(wl.cameras), 0)
    # warm-up
    for it in range(1, args.warmup + 1):
        v = schedule[it - 1]
        tr.step(it, wl.cameras[v], wl.images_u8[v])
    torch.cuda.synchronize()
    log(f"[ours] FP32 FMA probe: {measure_fp32_peak()}")
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

    # ---- the reference's precision: the float64 raster build through the
    # public render API (not the training step; reported beside it)
    api64 = api_render_timing(tr, wl, schedule[0], torch.float64)

    # ---- end-to-end through the public API: GT H2D from pinned host + loss D2H
    e2e = end_to_end(tr, wl, schedule, args)

    # ---- second regime: the same step after more training
    warm = warm_regime(tr, wl, schedule, args) if args.warm_iters > 0 else None

    # ---- CPU baseline: the reference path (oracle port) on this host
    cpu, parity = ((None, None) if args.no_cpu_baseline
                   else cpu_baseline(wl, args, schedule, cfg, scene_extent))

    # kernels per step, all ours (no library kernels on the path): the ncu
    # launch list of one config-3 step (profiles/r02_final/launches.md) --
    # preprocess, depth radix sort (5 passes x 3: upsweep, chunk scan with the
    # sums scanned by its last CTA, scatter) + tie fix, gather with live
    # counts and the rank inverse + one scan (2), live emission, tile radix
    # sort (2 x 3), offsets, heavy-first order (1), raster fwd, loss (3),
    # raster bwd, fused live fold + chain, Adam (+ the chunk items launch when
    # the image is chunked, config 2)
    launches_per_step = 36 + (1 if tr.r.chunks is not None and tr.r.chunks.chunk else 0)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic gyroid isosurface; GT = quantize8(raycast_isosurface) on the GPU (the reference dataset recipe, 8-bit codes)",
        "config": workload_config(args.config, n, res, len(wl.cameras)),
        "roofline": roof, "cpu_baseline": cpu, "parity": parity, "e2e": e2e, "clocks": clocks,
        "gpu_launches": launches_per_step * args.steps,
        "phases_ms": {k: round(v, 4) for k, v in phases.items()},
        "render_api_f64": api64,
        "pairs": counts,
        "warm": warm,
    }
    emit(line)


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
                "peak_source": fp32_peak_source(),
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


_FP32 = {}


def measure_fp32_peak() -> dict:
    """FP32 FMA-pipe throughput measured on this GPU now (isg_probe_ffma:
    8 independent FFMA chains per thread, 8 CTAs of 256 per SM): best of 10
    launches (burst) and the mean of 200 back-to-back launches (sustained,
    ~0.4 s, the state a kernel inside a long step runs in)."""
    import torch
    from paper_2509_05216_b200 import _lib as L
    blocks, iters = 148 * 8, 2048
    flops = blocks * 256 * iters * 16 * 8 * 2
    out = torch.empty(blocks, dtype=torch.float32, device="cuda")
    s = L.stream_ptr()
    fn = L.lib().isg_probe_ffma

    def launch():
        L.check(fn(blocks, iters, L.ptr(out), s), "isg_probe_ffma")

    launch()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
    ev[0].record()
    for k in range(10):
        launch()
        ev[k + 1].record()
    torch.cuda.synchronize()
    best = min(ev[k].elapsed_time(ev[k + 1]) for k in range(10))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(200):
        launch()
    b.record()
    torch.cuda.synchronize()
    mean = a.elapsed_time(b) / 200
    _FP32.update({"burst_tflops": flops / (best * 1e-3) / 1e12,
                  "sustained_tflops": flops / (mean * 1e-3) / 1e12})
    return dict(_FP32)


def fp32_peak():
    """The roofline denominator of the raster kernels: the measured sustained
    FFMA rate when bench.py has probed it, else 148 SM x 128 lanes x 2 x max
    clock."""
    if "sustained_tflops" in _FP32:
        return _FP32["sustained_tflops"]
    peaks, _ = read_peaks()
    mhz = peaks.get("sm_max_mhz", 1965.0)
    return 148 * 128 * 2 * mhz * 1e6 / 1e12


def fp32_peak_source() -> str:
    if "sustained_tflops" in _FP32:
        return ("measured in this run: isg_probe_ffma, mean of 200 back-to-back launches "
                f"(burst {_FP32['burst_tflops']:.2f} TFLOP/s)")
    return "FP32 FFMA peak 148 SM x 128 lanes x 2 x max SM clock (not measured)"


def api_render_timing(tr, wl, view, dtype, reps: int = 3):
    """Device time of one forward + backward render of `view` through the
    public API (project, sort_order, tile lists, raster forward / backward in
    `dtype`, the scratch fold and chain rule; rasterizer.render_forward /
    render_backward) on the trainer's current Gaussians."""
    import torch
    import paper_2509_05216_b200 as P
    cam = wl.cameras[view]
    res = wl.resolution
    cloud = tr.cloud
    dl = torch.full((res, res, 3), 1e-3, dtype=dtype, device=cloud.positions.device)

    def once():
        batch = P.project(cloud, cam)
        img, aux, order = P.render_forward(batch, res, res, dtype=dtype)
        return batch, aux, order

    batch, aux, order = once()
    P.render_backward(cloud, cam, batch, order, aux, dl)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    f = b = 0.0
    for _ in range(reps):
        torch.cuda.synchronize()
        ev[0].record()
        batch, aux, order = once()
        ev[1].record()
        P.render_backward(cloud, cam, batch, order, aux, dl)
        ev[2].record()
        torch.cuda.synchronize()
        f += ev[0].elapsed_time(ev[1]) / reps
        b += ev[1].elapsed_time(ev[2]) / reps
    return {"dtype": str(dtype).replace("torch.", ""), "forward_ms": round(f, 3),
            "backward_ms": round(b, 3), "images_per_s": round(1000.0 / (f + b), 2),
            "view": int(view), "note": "public render API (full lists, unmasked raster pair, "
            "host-synchronised sizes), no optimiser step: a precision reference, not the metric"}


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


def cpu_baseline(wl, args, schedule, cfg, scene_extent):
    """The oracle port of the reference path on this host's cores: one full
    training iteration of the same workload from the initial state on the
    schedule's first view (bounded sample), and -- from its outputs -- the
    parity of our first training step on the same view and state (a fresh
    Trainer): depth order and tile lists bit-exact, loss, gradients, Adam on
    our gradients bit-exact, post-step parameters vs the oracle's step."""
    import numpy as np
    import torch
    from oracle import oracle as O
    from oracle import train as T
    try:
        O.build()
        params, state, seen, gacc = host_state(wl.points, wl.log_scales)
        v = schedule[0]
        img = (wl.images_u8[v].cpu().numpy().astype(np.float64) / 255.0).astype(np.float32)
        ocfg = T.Config(iterations=cfg.iterations, eval_interval=0, seed=0)
        pre = {k: a.copy() for k, a in params.items()}
        t0 = time.perf_counter()
        oloss, det = T.iteration(params, state, seen, gacc, 1, 1, wl.cameras[v], img, ocfg,
                                 scene_extent)
        per = time.perf_counter() - t0
        cpu = {"value": 1.0 / per, "unit": UNIT, "cores": O.num_threads(), "kind": "port",
               "sample": f"1 training iteration of {args.config} ({wl.points.shape[0]} "
                         f"Gaussians, {wl.resolution}^2, view {v}) on the oracle (C, OpenMP)",
               "seconds": per, "cpu_model": cpu_model(), "host_cpus": os.cpu_count()}
    except Exception as exc:  # noqa: BLE001 -- report, never fail the bench line
        return ({"value": None, "unit": UNIT, "cores": None, "kind": "port",
                 "sample": f"failed: {exc!r}"}, None)
    return cpu, step_parity(wl, v, cfg, scene_extent, pre, params, oloss, det)


def _rel_l2(a, b):
    import numpy as np
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _max_rel(a, b):
    import numpy as np
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)) if b.size else 0.0


def step_parity(wl, v, cfg, scene_extent, pre, post, oloss, det):
    """Our first training step (Trainer.step, the timed launches) on view v
    from the initial state `pre` vs the oracle's iteration from the same state
    (loss `oloss`, details `det`, post-step parameters `post`); bars as in
    tests/test_scale_parity_gpu.py."""
    import numpy as np
    import torch
    import paper_2509_05216_b200 as P
    from oracle import oracle as O
    from paper_2509_05216_b200.engine import Trainer
    try:
        dev = wl.images_u8.device
        cloud = P.cloud_from_points(wl.points, wl.log_scales, 1, dev)
        tr = Trainer(cloud, wl.resolution, wl.resolution, cfg, scene_extent, dev)
        tr.r.keep_grads = True  # the parameter gradients, for the comparison below
        tr.step(1, wl.cameras[v], wl.images_u8[v])
        torch.cuda.synchronize()
        PN = P.PARAM_NAMES
        out = {"view": int(v), "state": "initial (iteration 1)"}
        got = float(tr.loss_dev[1])
        out["loss"] = got
        out["loss_oracle"] = oloss
        out["loss_rel"] = abs(got - oloss) / abs(oloss)
        r = tr.r
        m = int((r.rank_of >= 0).sum())
        out["depth_order_bitexact"] = bool(np.array_equal(r.order[:m].cpu().numpy(),
                                                          det["depth_order_rows"]))
        # the reference's full tile lists through the API path
        batch = P.project(cloud_from_host(pre, dev), wl.cameras[v])
        order = P.sort_order(batch)
        off, ent = P.build_tile_lists(batch.tile_min[order], batch.tile_max[order],
                                      np.arange(batch.tiles_x * batch.tiles_y, dtype=np.int32),
                                      batch.tiles_x, batch.tiles_y)
        out["tile_lists_bitexact"] = bool(np.array_equal(off.cpu().numpy(), det["offsets"]) and
                                          np.array_equal(ent.cpu().numpy(), det["entries"]))
        del batch, order, off, ent
        out["grad_rel_l2"] = {k: _rel_l2(tr.grads[k].cpu().numpy(), det["param_grads"][k])
                              for k in PN}
        out["grad_max_rel"] = {k: _max_rel(tr.grads[k].cpu().numpy(), det["param_grads"][k])
                               for k in PN}
        # Adam on our gradients == our post-step state (reference arithmetic)
        pa = {k: pre[k].copy() for k in PN}
        sa = {k: {"m": np.zeros_like(pre[k]), "v": np.zeros_like(pre[k])} for k in PN}
        O.adam_step(pa, {k: tr.grads[k].cpu().numpy() for k in PN}, sa, 1, det["lrs"])
        out["adam_bitexact_on_our_grads"] = all(
            np.array_equal(getattr(tr.cloud, k).cpu().numpy(), pa[k]) for k in PN)
        # vs the oracle's own step (float64 gradients)
        out["params_within_0.05lr"] = {}
        for k in PN:
            d = np.abs(getattr(tr.cloud, k).cpu().numpy().astype(np.float64)
                       - post[k].astype(np.float64))
            out["params_within_0.05lr"][k] = float(np.mean(d <= 0.05 * det["lrs"][k]))
        out["bars"] = ("order/lists/Adam bit-exact; loss rel <= 2e-5; grad rel L2 <= 1e-3; "
                       "params within 0.05 lr >= 99.9 %")
        out["pass"] = bool(out["depth_order_bitexact"] and out["tile_lists_bitexact"]
                           and out["adam_bitexact_on_our_grads"] and out["loss_rel"] <= 2e-5
                           and max(out["grad_rel_l2"].values()) <= 1e-3
                           and min(out["params_within_0.05lr"].values()) >= 0.999)
        del tr
        torch.cuda.empty_cache()
        return out
    except Exception as exc:  # noqa: BLE001
        return {"error": repr(exc)}


def cloud_from_host(params, dev):
    import torch
    import paper_2509_05216_b200 as P
    return P.GaussianCloud(*(torch.from_numpy(params[k]).to(dev) for k in P.PARAM_NAMES),
                           degree=1)


def run_dist(args, world: int, rank: int, local: int):
    """The sharded step on `world` GPUs, one process each (distributed.py):
    Gaussian shards + pixel row bands, splat and gradient all-to-all-v, SSIM
    halo, loss all-reduce.  value = world-wide images/s over K steps timed as
    the max over ranks of CUDA events on each rank's stream.  Each rank also
    reports its phase times and the roofline of its raster backward over its
    band's pair counts; rank 0 runs the CPU baseline and the step parity."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2509_05216_b200 import synthetic as S
    from paper_2509_05216_b200 import distributed as D
    from paper_2509_05216_b200.engine import PhaseTimer
    from paper_2509_05216_b200.gaussians import cloud_from_points
    from paper_2509_05216_b200.training import TrainConfig, TrainDataset, PointCloud, build_schedule
    dev = torch.device("cuda", local)
    # torchrun pins OMP_NUM_THREADS=1; the host side of the step runs slower that way
    torch.set_num_threads(max(1, (os.cpu_count() or 1) // max(world, 1)))
    say = log if rank == 0 else (lambda *a: None)
    wl = S.make_workload(args.config, dev, log=say, resolution=args.res)
    n = wl.points.shape[0]
    res = wl.resolution
    exchange = args.exchange
    try:
        comm = D.TorchComm(peers=exchange == "peer", height=res, width=res, device=dev)
    except Exception as exc:  # no symmetric memory / peer mapping on this box
        say(f"[dist] peer-store exchange unavailable ({type(exc).__name__}: {exc}); "
            "using point-to-point NCCL copies")
        exchange = f"nccl (peer unavailable: {type(exc).__name__})"
        comm = D.TorchComm(peers=False)
    cloud = cloud_from_points(wl.points, wl.log_scales, 1, dev)
    iters = args.warmup + args.steps
    cfg = TrainConfig(iterations=total_iterations(args), densify=False, eval_interval=0)
    ext = TrainDataset(wl.cameras, np.zeros((len(wl.cameras), 1, 1, 3)),
                       PointCloud(wl.points, wl.normals)).scene_extent
    (rs,), smap, part = D.make_ranks(cloud, res, res, cfg, ext, world, dev, only_rank=rank)
    del cloud
    schedule = build_schedule(cfg.iterations, len(wl.cameras), 0)
    for it in range(1, args.warmup + 1):
        v = schedule[it - 1]
        D.comm_step(rs, comm, wl.cameras[v], wl.images_u8[v], it)
    torch.cuda.synchronize()
    say(f"[dist] FP32 FMA probe (rank 0): {measure_fp32_peak()}")
    dist.barrier()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        dist.barrier()
        start.record()
        for it in range(args.warmup + 1, iters + 1):
            v = schedule[it - 1]
            D.comm_step(rs, comm, wl.cameras[v], wl.images_u8[v], it)
        stop.record()
        torch.cuda.synchronize()
        dist.barrier()
    ms = torch.tensor([start.elapsed_time(stop)], dtype=torch.float64, device=dev)
    comm.max_(ms)
    ms_per_step = float(ms[0]) / args.steps
    # per-rank roofline units of the next view, then one more step with
    # CUDA events between its phases (both untimed)
    v = schedule[iters]
    counts = D.comm_pair_counts(rs, comm, wl.cameras[v])
    timer = PhaseTimer()
    D.comm_step(rs, comm, wl.cameras[v], wl.images_u8[v], iters + 1, timer=timer)
    phases = {k: round(x, 4) for k, x in timer.phases().items()}
    flops = 13 * counts["I_b"] + 55 * counts["C"]
    bwd_ms = phases.get("raster_bwd", float("nan"))
    fp32 = fp32_peak()
    achieved = flops / (bwd_ms * 1e-3) / 1e12 if bwd_ms > 0 else None
    mine = {"rank": rank, "band_tile_rows": [rs.trow0, rs.trow1], "phases_ms": phases,
            "pairs": counts, "raster_bwd_tflops": achieved,
            "raster_bwd_frac": achieved / fp32 if achieved else None,
            "step_ms": sum(x for k, x in phases.items() if k != "begin")}
    per_rank = [None] * world
    dist.all_gather_object(per_rank, mine)
    say("[dist] per-rank phases (ms): " + "; ".join(
        f"r{r['rank']} " + ", ".join(f"{k} {x:.3f}" for k, x in r["phases_ms"].items())
        for r in per_rank))
    # end to end: each step's GT H2D from pinned host memory + loss D2H
    first = iters + 2
    host = torch.empty((args.steps,) + tuple(wl.images_u8.shape[1:]),
                       dtype=torch.uint8).pin_memory()
    for k in range(args.steps):
        host[k].copy_(wl.images_u8[schedule[first + k - 1]].cpu())
    gt = torch.empty_like(wl.images_u8[0])
    lh = torch.zeros(1, dtype=torch.float64).pin_memory()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(args.steps):
        it = first + k
        v = schedule[it - 1]
        gt.copy_(host[k], non_blocking=True)
        loss = D.comm_step(rs, comm, wl.cameras[v], gt, it)
        lh.copy_(loss, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        _ = float(lh[0])
    e1.record()
    torch.cuda.synchronize()
    ems = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    comm.max_(ems)
    cpu = parity = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu, parity = cpu_baseline(wl, args, schedule, cfg, ext)
    dist.barrier()
    if rank == 0:
        slow = max(per_rank, key=lambda r: r["phases_ms"].get("raster_bwd", 0.0))
        roof = {"kernel": "raster_bwd", "bound": "fp32", "achieved": slow["raster_bwd_tflops"],
                "peak": fp32, "unit": "TFLOP/s", "frac": slow["raster_bwd_frac"],
                "traffic": None, "rank": slow["rank"],
                "algorithmic": "13 I_b + 55 C flops over the rank's band (SURVEY 8d)",
                "peak_source": fp32_peak_source(),
                "per_rank": [{"rank": r["rank"], "achieved": r["raster_bwd_tflops"],
                              "frac": r["raster_bwd_frac"]} for r in per_rank]}
        line = {
            "metric": METRIC, "value": 1000.0 / ms_per_step, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic gyroid isosurface; GT = quantize8(raycast_isosurface) on the GPU (the reference dataset recipe, 8-bit codes)",
            "config": workload_config(args.config, n, res, len(wl.cameras)),
            "e2e": {"value": 1000.0 * args.steps / float(ems[0]), "unit": UNIT,
                    "h2d_bytes_per_step": int(gt.numel()), "d2h_bytes_per_step": 8},
            "clocks": clk.summary(), "gpu_launches": D.LAUNCHES_PER_STEP * args.steps,
            "roofline": roof, "cpu_baseline": cpu, "parity": parity,
            "exchange": exchange,
            "partition": {"bands_tile_rows": rs.part.band_rows, "initial": part.band_rows,
                          "canon_rows": part.canon_rows, "shard_sizes": smap.sizes,
                          "balance": rs.balance},
            "per_rank": per_rank,
        }
        emit(line)


def relaunch(args) -> int:
    """`bench.py --gpus N` outside torchrun: launch N ranks (one process per
    GPU) through torch.distributed.run on 127.0.0.1 and return its exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    log("[bench] launching: " + " ".join(cmd))
    return subprocess.call(cmd)


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
    ap.add_argument("--cpu-budget-s", type=float, default=120.0,
                    help="reference arm: stop timing iterations after this many seconds")
    ap.add_argument("--exchange", default=os.environ.get("ISOGS_EXCHANGE", "peer"),
                    choices=["peer", "nccl"],
                    help="sharded step's exchange: peer = NVLink stores from the pack / band "
                         "fold / forward kernels into symmetric-memory buffers; nccl = "
                         "point-to-point NCCL copies")
    ap.add_argument("--dist", action="store_true",
                    help="run the sharded engine even at N=1 (world 1)")
    args = ap.parse_args()
    _claim_stdout()
    if args.warmup < 3:
        log("[bench] warm-up raised to the required minimum of 3")
        args.warmup = 3
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
        rank = int(os.environ.get("RANK", "0"))
        return run_reference(args, world, rank)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    world, rank, local = dist_setup(args)
    if world != args.gpus and rank == 0:
        log(f"[bench] WORLD_SIZE={world} but --gpus {args.gpus}: reporting n_gpus={world}")
    if world > 1 or args.dist:
        run_dist(args, world, rank, local)
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
