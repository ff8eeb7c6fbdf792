"""Host issue time of one Trainer.step (wall clock around the call, no sync
inside except the step's own) vs its device time, at a config."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200 import synthetic as S
    from paper_2509_05216_b200.engine import Trainer
    from paper_2509_05216_b200.training import TrainConfig, TrainDataset, PointCloud, build_schedule
    cfgname = sys.argv[1] if len(sys.argv) > 1 else "config2"
    dev = torch.device("cuda", 0)
    nv = S.CONFIGS[cfgname][4]
    sched = build_schedule(30, nv, 0)
    wl = S.make_workload(cfgname, dev, view_ids=sched, log=lambda *x: None)
    ext = TrainDataset(wl.cameras, np.zeros((nv, 1, 1, 3)), PointCloud(wl.points, wl.normals)).scene_extent
    tr = Trainer(P.cloud_from_points(wl.points, wl.log_scales, 1, dev), wl.resolution,
                 wl.resolution, TrainConfig(iterations=30, densify=False), ext, dev)
    for it in range(1, 6):
        tr.step(it, wl.cameras[sched[it - 1]], wl.images_u8[it - 1])
    torch.cuda.synchronize()
    hs = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t_all = time.perf_counter()
    for it in range(6, 26):
        t0 = time.perf_counter()
        tr.step(it, wl.cameras[sched[it - 1]], wl.images_u8[it - 1])
        hs.append((time.perf_counter() - t0) * 1e3)
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t_all) * 1e3 / 20
    print(f"{cfgname}: host per step {np.mean(hs):.3f} ms (median {np.median(hs):.3f}), "
          f"device {e0.elapsed_time(e1) / 20:.3f} ms/step, wall {wall:.3f}")


if __name__ == "__main__":
    main()
