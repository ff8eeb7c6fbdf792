"""Per-rank device time of the sharded step at W ranks, emulated on one GPU.

W ranks' phases run in sequence on one B200 (distributed.emulated_step), each
phase of each rank bracketed by CUDA events, so every rank's compute is what
its own GPU would spend; the exchanges (device copies here) are replaced by
their byte counts.  The projected step time of a real W-GPU run is
  max over ranks of (rank compute) + splat exchange + gradient exchange
  + host sync latency,
with the exchanges at `--link-gbs` per direction per GPU (NVLink 5 through
NVSwitch: 900 GB/s nominal; a conservative achieved figure by default).

    python tools/emulated_ranks.py --config config3 --workers 8 > profiles/.../emul_w8.json
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="config3")
    ap.add_argument("--res", type=int, default=None)
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--warm", type=int, default=24)
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--link-gbs", type=float, default=600.0)
    ap.add_argument("--sync-us", type=float, default=60.0,
                    help="host round trip of the one sync per step (measured at W=1)")
    a = ap.parse_args()
    import torch
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200 import distributed as D
    from paper_2509_05216_b200 import synthetic as S
    from paper_2509_05216_b200.training import TrainConfig, TrainDataset, PointCloud, build_schedule
    dev = torch.device("cuda", 0)
    nv = S.CONFIGS[a.config][4]
    total = a.warm + a.steps
    sched = build_schedule(total, nv, 0)
    wl = S.make_workload(a.config, dev, view_ids=sched, resolution=a.res,
                         log=lambda *x: print(*x, file=sys.stderr))
    ext = TrainDataset(wl.cameras, np.zeros((nv, 1, 1, 3)),
                       PointCloud(wl.points, wl.normals)).scene_extent
    cfg = TrainConfig(iterations=total, densify=False, eval_interval=0)
    cloud = P.cloud_from_points(wl.points, wl.log_scales, 1, dev)
    ranks, smap, part = D.make_ranks(cloud, wl.resolution, wl.resolution, cfg, ext, a.workers, dev)
    del cloud
    W = a.workers
    for it in range(1, a.warm + 1):
        D.emulated_step(ranks, wl.cameras[sched[it - 1]], wl.images_u8[it - 1], it)
    torch.cuda.synchronize()
    per_step = []
    for it in range(a.warm + 1, total + 1):
        timers = [D.SpanTimer() for _ in range(W)]
        D.emulated_step(ranks, wl.cameras[sched[it - 1]], wl.images_u8[it - 1], it, timers=timers)
        ph = [t.phases() for t in timers]
        ex = []
        for r in ranks:
            me = r.rank
            splat_out = sum(c for d, c in enumerate(r.send_cnt) if d != me) * 72
            splat_in = sum(c for s_, c in enumerate(r.recv_cnt) if s_ != me) * 72
            grad_out = sum(c for s_, c in enumerate(r.gsend_cnt) if s_ != me) * 72
            grad_in = sum(c for d, c in enumerate(r.grecv_cnt) if d != me) * 72
            ex.append({"splat_bytes": max(splat_out, splat_in), "grad_bytes": max(grad_out, grad_in)})
        per_step.append({"phases": ph, "exchange": ex, "bands": list(ranks[0].part.band_rows)})
    # aggregate
    names = sorted({k for s in per_step for p in s["phases"] for k in p})
    mean_ph = [{k: float(np.mean([s["phases"][r].get(k, 0.0) for s in per_step])) for k in names}
               for r in range(W)]
    comp = [float(np.mean([sum(s["phases"][r].values()) for s in per_step])) for r in range(W)]
    step_max = [max(sum(s["phases"][r].values()) for r in range(W)) for s in per_step]
    bw = a.link_gbs * 1e9
    xs = [max(e["splat_bytes"] for e in s["exchange"]) / bw * 1e3 for s in per_step]
    xg = [max(e["grad_bytes"] for e in s["exchange"]) / bw * 1e3 for s in per_step]
    proj = [m + p + g + a.sync_us * 1e-3 for m, p, g in zip(step_max, xs, xg)]
    raster = [[s["phases"][r].get("bin_render", 0) + s["phases"][r].get("backward_fold", 0)
               for r in range(W)] for s in per_step]
    out = {
        "workload": a.config, "resolution": wl.resolution, "workers": W, "steps_timed": a.steps,
        "after_warm_steps": a.warm, "canon_rows": part.canon_rows,
        "bands_final": ranks[0].part.band_rows, "balance": ranks[0].balance,
        "per_rank_mean_phases_ms": mean_ph, "per_rank_compute_ms": comp,
        "band_compute_max_over_mean": float(np.mean([max(x) / np.mean(x) for x in raster])),
        "step_compute_max_ms": float(np.mean(step_max)),
        "exchange_ms": {"splats": float(np.mean(xs)), "grads": float(np.mean(xg)),
                        "link_gbs": a.link_gbs},
        "host_sync_ms": a.sync_us * 1e-3,
        "projected_step_ms_mean": float(np.mean(proj)),
        "projected_step_ms": float(np.median(proj)),
        "projected_images_per_s": 1000.0 / float(np.median(proj)),
        "note": "emulated on one B200: each rank's phases timed alone (CUDA events); exchanges "
                "projected from their byte counts; the projection is the median step (a step "
                "that grows a buffer pays a one-off allocation inside a timed phase)",
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
