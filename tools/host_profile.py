"""Host cost of the training step: per step, the host time spent issuing
work (wall minus the time blocked in the step's one synchronisation), for
the single-GPU engine and for one rank of the sharded step (emulated W
ranks: each rank's host work is what its own process would do), plus a
cProfile of the issuing code.

    python tools/host_profile.py config2 [W]
"""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200 import distributed as D
    from paper_2509_05216_b200 import synthetic as S
    from paper_2509_05216_b200.engine import Trainer
    from paper_2509_05216_b200.training import TrainConfig, TrainDataset, PointCloud, build_schedule
    cfgname = sys.argv[1] if len(sys.argv) > 1 else "config2"
    W = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    dev = torch.device("cuda", 0)
    nv = S.CONFIGS[cfgname][4]
    sched = build_schedule(60, nv, 0)
    wl = S.make_workload(cfgname, dev, view_ids=sched, log=lambda *x: None)
    ext = TrainDataset(wl.cameras, np.zeros((nv, 1, 1, 3)), PointCloud(wl.points, wl.normals)).scene_extent
    cfg = TrainConfig(iterations=60, densify=False, eval_interval=0)
    wait = [0.0]
    orig = torch.cuda.Stream.synchronize

    def timed_sync(self):
        t = time.perf_counter()
        orig(self)
        wait[0] += time.perf_counter() - t
    torch.cuda.Stream.synchronize = timed_sync

    def measure(step, its):
        torch.cuda.synchronize()
        wait[0] = 0.0
        t0 = time.perf_counter()
        for it in its:
            step(it)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        n = len(its)
        return (t1 - t0 - wait[0]) * 1e3 / n, wait[0] * 1e3 / n

    tr = Trainer(P.cloud_from_points(wl.points, wl.log_scales, 1, dev), wl.resolution,
                 wl.resolution, cfg, ext, dev)
    step1 = lambda it: tr.step(it, wl.cameras[sched[it - 1]], wl.images_u8[it - 1])
    for it in range(1, 6):
        step1(it)
    issue, blocked = measure(step1, range(6, 26))
    print(f"{cfgname} single GPU: host issue {issue:.3f} ms/step, blocked in sync {blocked:.3f}")
    pr = cProfile.Profile()
    pr.enable()
    for it in range(26, 36):
        step1(it)
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(22)
    del tr
    torch.cuda.empty_cache()

    ranks, _, _ = D.make_ranks(P.cloud_from_points(wl.points, wl.log_scales, 1, dev),
                               wl.resolution, wl.resolution, cfg, ext, W, dev)
    stepW = lambda it: D.emulated_step(ranks, wl.cameras[sched[it - 1]], wl.images_u8[it - 1],
                                       it, peers=True)
    for it in range(1, 6):
        stepW(it)
    issue, blocked = measure(stepW, range(6, 16))
    print(f"{cfgname} sharded W={W} (emulated, peer stores): host issue per rank "
          f"{issue / W:.3f} ms/step (all ranks {issue:.3f}), blocked {blocked:.3f}")
    pr = cProfile.Profile()
    pr.enable()
    for it in range(16, 21):
        stepW(it)
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(22)


if __name__ == "__main__":
    main()
