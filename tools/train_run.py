"""End-to-end training run of a BASELINE workload on one GPU through the public
API (run_training, the reference's default TrainConfig: densify/prune every
100 iterations from 500 to iters/2, dense Adam), with evaluation (PSNR/SSIM
over every view, the reference's _evaluate) before and after training.

    python tools/train_run.py --config config4 --iters 2000 > gpurun_out/train_config4.json

Prints one JSON line: Gaussians before/after, training wall (eval excluded,
TrainReport.total_wall_s), images/s, loss trace summary and the eval records.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="config4")
    ap.add_argument("--iters", type=int, default=2000)
    ap.add_argument("--eval-interval", type=int, default=0)
    a = ap.parse_args()
    import torch
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200 import synthetic as S

    dev = torch.device("cuda", 0)
    t0 = time.time()
    wl = S.make_workload(a.config, dev, log=lambda *x: print(*x, file=sys.stderr))
    setup_s = time.time() - t0
    ds = P.TrainDataset(cameras=wl.cameras, images=wl.images_u8,
                        points=P.PointCloud(wl.points, wl.normals))
    init = P.cloud_from_points(wl.points, wl.log_scales, 1, dev)
    n0 = init.count
    cfg = P.TrainConfig(iterations=a.iters, eval_interval=a.eval_interval, seed=0)
    t1 = time.time()
    cloud, rep = P.run_training(ds, cfg, workers=1, init_cloud=init, evaluate=True)
    torch.cuda.synchronize()
    total_s = time.time() - t1
    losses = rep.iteration_losses
    out = {
        "workload": a.config, "gaussians_init": n0, "gaussians_final": cloud.count,
        "resolution": wl.resolution, "views": len(wl.cameras), "iterations": a.iters,
        "config": {k: getattr(cfg, k) for k in ("densify", "densify_interval", "densify_start",
                                                 "grad_threshold", "opacity_prune", "seed")},
        "train_wall_s": rep.total_wall_s, "images_per_s": a.iters / rep.total_wall_s,
        "run_wall_s_incl_eval": total_s, "setup_s": setup_s,
        "loss_first10_mean": sum(losses[:10]) / min(10, len(losses)),
        "loss_last10_mean": sum(losses[-10:]) / min(10, len(losses)),
        "records": [{"iteration": r.iteration, "gaussians": r.gaussians, "loss": r.loss,
                     "psnr": r.psnr, "ssim": r.ssim} for r in rep.records],
        "device": torch.cuda.get_device_name(0),
        "note": "synthetic gyroid isosurface, GT = quantize8(raycast_isosurface) on the GPU; "
                "wall includes densify steps, excludes evaluation",
    }
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
