"""Row-band load balance of the pixel partition, measured.

For a workload, renders `--views` orbit views on one GPU with the per-pixel
pair counters (n_iter = pairs the forward iterates, n_last = the backward's
last contributor index) and takes the per-tile-row raster cost
I_f + I_b.  For each canonical block height (canon_rows: bands must be
unions of whole blocks) and each GPU count W it reports the band cost
max/mean of
  * equal bands (the same number of blocks per band),
  * static cost-balanced bands (cut once from the mean cost over the views),
  * per-view optimal bands (the best contiguous cut of each view's own cost),
  * per-view bands cut from a predictor known before routing (the view's
    tile entries per tile row, each tile's count capped at CAPS),
and the mean number of gradient block records per visible splat (the
size of the gradient exchange grows with it).

    python tools/band_balance.py --config config3 --views 32 > profiles/.../band_balance.json
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


CAPS = (1e9, 100, 200, 400, 800, 1600)


def best_cuts(w: np.ndarray, parts: int) -> list:
    """Contiguous split of the block costs `w` into `parts` non-empty groups
    minimising the maximum group cost (DP; blocks <= a few hundred)."""
    b = len(w)
    pre = np.concatenate([[0.0], np.cumsum(w)])
    inf = float("inf")
    dp = np.full((parts + 1, b + 1), inf)
    arg = np.zeros((parts + 1, b + 1), dtype=np.int64)
    dp[0, 0] = 0.0
    for p in range(1, parts + 1):
        for j in range(p, b + 1):
            best, bi = inf, -1
            for i in range(p - 1, j):
                c = max(dp[p - 1, i], pre[j] - pre[i])
                if c < best:
                    best, bi = c, i
            dp[p, j], arg[p, j] = best, bi
    cuts = [b]
    j = b
    for p in range(parts, 0, -1):
        j = int(arg[p, j])
        cuts.append(j)
    return cuts[::-1]


def ratio(w: np.ndarray, cuts: list) -> float:
    s = np.array([w[cuts[k]:cuts[k + 1]].sum() for k in range(len(cuts) - 1)])
    return float(s.max() / s.mean())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="config3")
    ap.add_argument("--res", type=int, default=None)
    ap.add_argument("--views", type=int, default=32)
    a = ap.parse_args()
    import torch
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200 import synthetic as S
    from paper_2509_05216_b200.engine import Rasterizer
    dev = torch.device("cuda", 0)
    nv_all = S.CONFIGS[a.config][4]
    ids = [int(v) for v in np.linspace(0, nv_all - 1, a.views).round()]
    wl = S.make_workload(a.config, dev, view_ids=ids[:1], resolution=a.res,
                         log=lambda *x: print(*x, file=sys.stderr))
    res = wl.resolution
    cloud = P.cloud_from_points(wl.points, wl.log_scales, 1, dev)
    r = Rasterizer(cloud.count, res, res, dev)
    r.use_cmask = False
    rows = (res + 15) // 16
    costs = []
    proxies = []
    spans = {}
    for v in ids:
        r.n_contrib_out = torch.zeros((res, res), dtype=torch.int32, device=dev)
        r.n_iter_out = torch.zeros((res, res), dtype=torch.int32, device=dev)
        ctx = r.forward(cloud, wl.cameras[v])
        per_px = (r.n_iter_out.to(torch.int64) + r.n_last.to(torch.int64))
        row = per_px.sum(dim=1).cpu().numpy()
        pad = np.zeros(rows * 16, dtype=np.float64)
        pad[:res] = row
        costs.append(pad.reshape(rows, 16).sum(axis=1))
        # predictor available before routing: tile entries per tile row
        off = r.offsets.cpu().numpy().astype(np.int64)
        e_tile = np.diff(off).reshape(rows, -1).astype(np.float64)
        proxies.append(np.stack([np.minimum(e_tile, cap).sum(axis=1) for cap in CAPS]))
        rect = r.rect_sorted[:ctx.m].cpu().numpy()
        for canon in (1, 2, 4, 8):
            nb = rect[:, 3] // canon - rect[:, 1] // canon + 1
            spans.setdefault(canon, []).append(float(nb.mean()))
    costs = np.array(costs)  # (views, tile rows)
    proxies = np.array(proxies)
    out = {"workload": a.config, "resolution": res, "views": ids, "tile_rows": rows,
           "cost": "I_f + I_b per tile row (pairs iterated by the forward + the backward's "
                   "last-contributor index), full reference lists", "by_canon": {}}
    for canon in (1, 2, 4, 8):
        nbk = (rows + canon - 1) // canon
        blk = np.zeros((len(ids), nbk))
        for k in range(nbk):
            blk[:, k] = costs[:, k * canon:(k + 1) * canon].sum(axis=1)
        mean_w = blk.mean(axis=0)
        pblk = np.zeros((len(ids), len(CAPS), nbk))
        for k in range(nbk):
            pblk[:, :, k] = proxies[:, :, k * canon:(k + 1) * canon].sum(axis=2)
        entry = {"blocks": nbk, "block_records_per_splat": float(np.mean(spans[canon]))}
        for W in (2, 4, 8):
            if nbk < W:
                continue
            eq = [round(k * nbk / W) for k in range(W + 1)]
            st = best_cuts(mean_w, W)
            entry[f"W{W}"] = {
                "equal": float(np.mean([ratio(c, eq) for c in blk])),
                "static_balanced": float(np.mean([ratio(c, st) for c in blk])),
                "per_view_optimal": float(np.mean([ratio(c, best_cuts(c, W)) for c in blk])),
                "per_view_entries_cut": {str(cap): float(np.mean([
                    ratio(c, best_cuts(p[q], W)) for c, p in zip(blk, pblk)]))
                    for q, cap in enumerate(CAPS)},
                "static_cuts_blocks": st,
            }
        out["by_canon"][str(canon)] = entry
    print(json.dumps(out))


if __name__ == "__main__":
    main()
