"""Small driver for ncu / compute-sanitizer: a few training steps of a
synthetic workload with few GT views (so kernel-name filters stay simple).

    python tools/profile_step.py --config config2 --views 4 --steps 2
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="config2")
    ap.add_argument("--views", type=int, default=4)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--points", type=int, default=None)
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200 import synthetic as S
    from paper_2509_05216_b200.engine import Trainer
    from paper_2509_05216_b200.training import TrainConfig
    dev = torch.device("cuda", 0)
    wl = S.make_workload(args.config, dev, views=args.views, max_points=args.points,
                         log=lambda *a: print(*a, file=sys.stderr))
    cloud = P.cloud_from_points(wl.points, wl.log_scales, 1, dev)
    cfg = TrainConfig(iterations=args.steps, densify=False)
    tr = Trainer(cloud, wl.resolution, wl.resolution, cfg, 300.0, dev)
    for it in range(1, args.steps + 1):
        v = (it - 1) % len(wl.cameras)
        tr.step(it, wl.cameras[v], wl.images_u8[v])
    torch.cuda.synchronize()
    print("losses", tr.loss_dev[1:args.steps + 1].tolist())


if __name__ == "__main__":
    main()
