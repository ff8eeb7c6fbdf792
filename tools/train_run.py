"""End-to-end training run of a BASELINE workload on one GPU through the public
API (run_training, the reference's default TrainConfig: densify/prune every
100 iterations from 500 to iters/2, dense Adam), with evaluation (PSNR/SSIM
over every view, the reference's _evaluate) before and after training.

    python tools/train_run.py --config config4 --iters 2000 > gpurun_out/train_config4.json
    python tools/train_run.py --config config4 --workers 4   # 4 GPUs: relaunches under torchrun

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
    ap.add_argument("--workers", type=int, default=1,
                    help="GPUs (one process each, the sharded engine; relaunched "
                         "through torch.distributed.run when WORLD_SIZE is unset)")
    a = ap.parse_args()
    if a.workers > 1 and "WORLD_SIZE" not in os.environ:
        import socket
        import subprocess
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        sys.exit(subprocess.call([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                  f"--nproc-per-node={a.workers}", "--master-addr", "127.0.0.1",
                                  "--master-port", str(port), os.path.abspath(__file__)]
                                 + sys.argv[1:]))
    import torch
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200 import synthetic as S

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if a.workers > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    t0 = time.time()
    wl = S.make_workload(a.config, dev, log=lambda *x: print(*x, file=sys.stderr))
    setup_s = time.time() - t0
    ds = P.TrainDataset(cameras=wl.cameras, images=wl.images_u8,
                        points=P.PointCloud(wl.points, wl.normals))
    init = P.cloud_from_points(wl.points, wl.log_scales, 1, dev)
    n0 = init.count
    cfg = P.TrainConfig(iterations=a.iters, eval_interval=a.eval_interval, seed=0)
    t1 = time.time()
    cloud, rep = P.run_training(ds, cfg, workers=a.workers, init_cloud=init, evaluate=True)
    torch.cuda.synchronize()
    total_s = time.time() - t1
    if a.workers > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
        if rank != 0:
            return
    losses = rep.iteration_losses
    out = {
        "workload": a.config, "workers": a.workers, "gaussians_init": n0, "gaussians_final": cloud.count,
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
