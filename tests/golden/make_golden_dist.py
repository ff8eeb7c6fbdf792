"""Golden fixtures of the reference's host-side data-plane helpers
(rebalance, route_splats), made by running the unmodified reference:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_dist.py

Writes tests/golden/dataplane.npz: seeded shard maps with their rebalance
plans and resulting lists, and seeded splat spans with their round-robin
per-worker lists (as gaussian indices in list order)."""

from __future__ import annotations

import os

import numpy as np

from isosplat import distributed as D
from isosplat.rasterizer import ProjectedSplat

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(11)
    out = {}
    # rebalance: random uneven contiguous-ish shard maps
    for case in range(6):
        w = int(rng.integers(2, 6))
        n = int(rng.integers(w, 60))
        perm = rng.permutation(n)
        cuts = np.sort(rng.choice(np.arange(1, n), size=w - 1, replace=False))
        lists = [np.sort(p) for p in np.split(perm, cuts)]
        smap = D.ShardMap.from_lists(lists, n)
        plan, new = D.rebalance(smap, smap.sizes)
        out[f"rb{case}_n"] = np.array(n)
        out[f"rb{case}_owner"] = smap.owner
        out[f"rb{case}_plan"] = np.array(plan, dtype=np.int64).reshape(-1, 3)
        out[f"rb{case}_new_owner"] = new.owner
    # route_splats: random spans over a 7 x 5 tile grid, 3 workers round-robin
    part = D.partition_pixels(7 * 16, 5 * 16, 16, 3)
    spl = []
    for i in range(40):
        x0, y0 = int(rng.integers(0, 7)), int(rng.integers(0, 5))
        x1, y1 = int(rng.integers(x0, 7)), int(rng.integers(y0, 5))
        depth = float(rng.choice([1.0, 2.0, 3.0]))  # ties break on the index
        spl.append(ProjectedSplat(gaussian_index=int(rng.integers(0, 1000)), mean2d=np.zeros(2),
                                  cov2d=np.zeros(3), depth=depth, color=np.zeros(3), opacity=0.5,
                                  tile_span=((x0, y0), (x1, y1))))
    lists = D.route_splats(spl, part)
    out["rs_spans"] = np.array([[s.tile_span[0][0], s.tile_span[0][1], s.tile_span[1][0],
                                 s.tile_span[1][1]] for s in spl], dtype=np.int32)
    out["rs_depth"] = np.array([s.depth for s in spl])
    out["rs_index"] = np.array([s.gaussian_index for s in spl], dtype=np.int64)
    out["rs_assignment"] = part.assignment
    for w, lst in enumerate(lists):
        out[f"rs_list{w}"] = np.array([s.gaussian_index for s in lst], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "dataplane.npz"), **out)
    print("wrote dataplane.npz")


if __name__ == "__main__":
    main()
