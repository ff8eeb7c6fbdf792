"""Diagnostic: how the forward's contribution masks split between the
backward's two 16x8 halves (config3 view 0): entries kept by the top half,
the bottom half, both, and the per-quadrant totals.

    python tools/cmask_stats.py [--config config3]
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def popc(x):
    import torch
    x = x.to(torch.int64) & 0xFFFFFFFF
    c = torch.zeros_like(x)
    for b in range(32):
        c += (x >> b) & 1
    return int(c.sum())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="config3")
    a = ap.parse_args()
    import numpy as np
    import torch
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200 import synthetic as S
    from paper_2509_05216_b200.engine import Trainer
    from paper_2509_05216_b200.training import TrainConfig
    dev = torch.device("cuda", 0)
    wl = S.make_workload(a.config, dev, views=4)
    cloud = P.cloud_from_points(wl.points, wl.log_scales, 1, dev)
    ext = P.TrainDataset(wl.cameras, np.zeros((len(wl.cameras), 1, 1, 3)),
                         P.PointCloud(wl.points, wl.normals)).scene_extent
    tr = Trainer(cloud, wl.resolution, wl.resolution, TrainConfig(iterations=1), ext, dev)
    # zeroed up front: words of batches a quadrant never reached stay 0
    tr.r.cmask = torch.zeros(4 * (100_000_000 // 32 + tr.r.n_tiles + 1), dtype=torch.int32, device=dev)
    ctx = tr.r.forward(tr.cloud, wl.cameras[0])
    torch.cuda.synchronize()
    e = ctx.e
    cm = tr.r.cmask[:4 * (e // 32 + tr.r.n_tiles + 1)].view(-1, 4)
    q = [cm[:, i] for i in range(4)]
    h0, h1 = q[0] | q[1], q[2] | q[3]
    k0, k1 = popc(h0), popc(h1)
    both, uniq = popc(h0 & h1), popc(h0 | h1)
    print(f"E={e} entries; kept: top {k0}, bottom {k1}, sum {k0 + k1} (entry-warps), "
          f"unique {uniq} ({100 * uniq / e:.1f}% of E), both halves {both} "
          f"({100 * both / max(uniq, 1):.1f}% of unique)")
    print("per quadrant:", [popc(x) for x in q])


if __name__ == "__main__":
    main()
