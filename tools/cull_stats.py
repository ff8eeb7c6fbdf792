"""Diagnostic: how many (pixel, entry) visits the raster loops make under
different culling granularities (sub-box of a 16x16 tile that one warp walks
an entry list for).  Counts, for each granularity (bx, by), the entries of
each tile that (a) can reach alpha >= 1/255 somewhere in the sub-box
(the same exact box test as raster_f32.cu:box_dead) and (b) lie before the
sub-box's last contributor (n_last), times the sub-box pixel count.

    python tools/cull_stats.py --config config3
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def box_dead(mx, my, a, b, c, thr, x0, y0, ex, ey):
    import torch
    lx = x0 - mx
    hx = lx + ex
    ly = y0 - my
    hy = ly + ey
    inside = (lx <= 0) & (hx >= 0) & (ly <= 0) & (hy >= 0)
    q = torch.full_like(mx, float("inf"))
    for d0 in (lx, hx):
        d1 = torch.clamp(-b * d0 / c, min=ly, max=hy)
        q = torch.minimum(q, a * d0 * d0 + 2 * b * d0 * d1 + c * d1 * d1)
    for e1 in (ly, hy):
        e0 = torch.clamp(-b * e1 / a, min=lx, max=hx)
        q = torch.minimum(q, a * e0 * e0 + 2 * b * e0 * e1 + c * e1 * e1)
    mdx = torch.maximum(lx.abs(), hx.abs())
    mdy = torch.maximum(ly.abs(), hy.abs())
    scale = a * mdx * mdx + 2 * b.abs() * mdx * mdy + c * mdy * mdy
    dead = -0.5 * q < thr - (1e-3 + 1e-5 * scale)
    return (dead & ~inside) | (thr > 0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="config3")
    ap.add_argument("--views", type=int, default=2)
    args = ap.parse_args()
    import numpy as np
    import torch
    import torch.nn.functional as F
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200 import synthetic as S
    from paper_2509_05216_b200.engine import Rasterizer
    dev = torch.device("cuda", 0)
    wl = S.make_workload(args.config, dev, views=args.views)
    cloud = P.cloud_from_points(wl.points, wl.log_scales, 1, dev)
    res = wl.resolution
    r = Rasterizer(cloud.count, res, res, dev)
    ctx = r.forward(cloud, wl.cameras[0])
    e = ctx.e
    off = r.offsets.long()
    ent = r.entries[:e].long()
    tiles = torch.repeat_interleave(torch.arange(r.n_tiles, device=dev), off[1:] - off[:-1])
    j = torch.arange(e, device=dev) - off[tiles]
    f = r.feat_sorted[ent]
    mx, my, a, b, c, op = f[:, 0], f[:, 1], f[:, 2], f[:, 3], f[:, 4], f[:, 5]
    thr = torch.where(op > 0, -torch.log(255.0 * op.clamp_min(1e-30)) - 1e-3,
                      torch.ones_like(op))
    ty, tx = tiles // r.tiles_x, tiles % r.tiles_x
    nl = r.n_last.float()[None, None]
    print(f"E={e} P={res * res} tiles={r.n_tiles}")
    base = None
    for bx, by in ((16, 16), (16, 8), (8, 16), (8, 8), (8, 4), (4, 8), (4, 4)):
        ml = F.max_pool2d(nl, (by, bx)).long()[0, 0]  # (H/by, W/bx)
        visits = 0
        reach = 0
        for sy in range(16 // by):
            for sx in range(16 // bx):
                x0 = (tx * 16 + sx * bx).float()
                y0 = (ty * 16 + sy * by).float()
                dead = box_dead(mx, my, a, b, c, thr, x0, y0, float(bx - 1), float(by - 1))
                lim = ml[ty * (16 // by) + sy, tx * (16 // bx) + sx]
                live = (~dead) & (j < lim)
                visits += int(live.sum()) * bx * by
                reach += int((~dead).sum()) * bx * by
        if base is None:
            base = visits
        print(f"box {bx:2d}x{by:2d}: pixel-visits {visits / 1e9:.3f}e9 ({visits / base:.3f} of tile), "
              f"per px {visits / (res * res):.1f}; reachable ignoring n_last {reach / 1e9:.3f}e9")


if __name__ == "__main__":
    main()
