"""Host-side issue time vs device time of the sharded step's phases at W
ranks (emulated on one GPU): per phase, the host wall time to issue every
rank's launches and the device time (CUDA events) they take.  A phase whose
host time exceeds its device time is launch-bound.

    python tools/host_overhead.py --config config3 --workers 8
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="config3")
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--steps", type=int, default=6)
    a = ap.parse_args()
    import numpy as np
    import torch
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200 import distributed as D
    from paper_2509_05216_b200 import synthetic as S
    from paper_2509_05216_b200.training import TrainConfig, TrainDataset, PointCloud, build_schedule
    dev = torch.device("cuda", 0)
    nv = S.CONFIGS[a.config][4]
    sched = build_schedule(a.steps + 4, nv, 0)
    wl = S.make_workload(a.config, dev, view_ids=sched, log=lambda *x: None)
    ext = TrainDataset(wl.cameras, np.zeros((nv, 1, 1, 3)), PointCloud(wl.points, wl.normals)).scene_extent
    cfg = TrainConfig(iterations=a.steps + 4, densify=False, eval_interval=0)
    cloud = P.cloud_from_points(wl.points, wl.log_scales, 1, dev)
    ranks, _, _ = D.make_ranks(cloud, wl.resolution, wl.resolution, cfg, ext, a.workers, dev)
    for it in range(1, 5):
        D.emulated_step(ranks, wl.cameras[sched[it - 1]], wl.images_u8[it - 1], it)
    torch.cuda.synchronize()
    host = {}
    dev_t = {}
    orig = {}
    names = ["phase_plan", "phase_sizes", "phase_pack", "phase_render", "phase_loss",
             "phase_backward", "phase_update"]
    for nm in names:
        orig[nm] = getattr(D.RankStep, nm)

        def wrap(self, *args, _nm=nm, **kw):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            t0 = time.perf_counter()
            out = orig[_nm](self, *args, **kw)
            host[_nm] = host.get(_nm, 0.0) + (time.perf_counter() - t0) * 1e3
            e1.record()
            dev_t.setdefault(_nm, []).append((e0, e1))
            return out
        setattr(D.RankStep, nm, wrap)
    for it in range(5, 5 + a.steps):
        D.emulated_step(ranks, wl.cameras[sched[it - 1]], wl.images_u8[it - 1], it)
    torch.cuda.synchronize()
    out = {}
    for nm in names:
        d = sum(e0.elapsed_time(e1) for e0, e1 in dev_t.get(nm, []))
        out[nm] = {"host_ms_per_rank_step": host.get(nm, 0) / (a.steps * a.workers),
                   "device_ms_per_rank_step": d / (a.steps * a.workers)}
    print(json.dumps({"config": a.config, "workers": a.workers, "phases": out}))


if __name__ == "__main__":
    main()
