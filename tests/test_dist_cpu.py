"""CPU tests of the multi-GPU host layer: partitions, routing, protocol
checks and the collectives (TorchComm) with world_size 2 over gloo."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_05216_b200 import distributed as D


def test_partition_gaussians_matches_reference_rules():
    smap = D.partition_gaussians(10, 3)
    assert smap.sizes == [4, 3, 3]
    assert smap.starts == [0, 4, 7, 10]
    np.testing.assert_array_equal(smap.lists[1], [4, 5, 6])
    smap = D.partition_gaussians(4_000_000, 4)
    assert smap.sizes == [1_000_000] * 4
    with pytest.raises(ValueError):
        D.partition_gaussians(5, 0)


@pytest.mark.parametrize("workers", [1, 2, 3, 4, 8])
def test_row_bands_are_unions_of_canonical_blocks(workers):
    part = D.partition_pixels(2048, 2048, 16, workers)
    assert part.band_rows[0] == 0 and part.band_rows[-1] == part.tiles_y
    for w in range(workers):
        assert part.band_rows[w] % part.canon_rows == 0
        assert part.band_rows[w + 1] > part.band_rows[w]
    a = part.assignment
    assert a.shape == (128 * 128,)
    assert (np.diff(a) >= 0).all()
    assert sorted(set(a.tolist())) == list(range(workers))


def test_row_bands_need_enough_blocks():
    with pytest.raises(ValueError):
        D.partition_pixels(64, 64, 16, 3)  # 4 tile rows = 2 blocks of 2
    part = D.partition_pixels(64, 64, 16, 4, canon_rows=1)
    assert part.band_rows == [0, 1, 2, 3, 4]


def test_cost_weighted_bands():
    part = D.partition_pixels(2048, 2048, 16, 2, weights=[40] + [1] * 63)
    assert part.band_rows[1] < 64  # the heavy first block pulls the cut up
    with pytest.raises(ValueError):
        D.partition_pixels(2048, 2048, 16, 2, weights=[1] * 16)


def test_minmax_cuts_is_optimal():
    import itertools
    rng = np.random.default_rng(0)
    for _ in range(300):
        b = int(rng.integers(2, 11))
        p = int(rng.integers(1, b + 1))
        w = rng.random(b) * (rng.random(b) < 0.8)
        c = D.minmax_cuts(w, p)
        assert c[0] == 0 and c[-1] == b and all(c[k] < c[k + 1] for k in range(p))
        best = min(max(w[a:e].sum() for a, e in zip((0,) + cs, cs + (b,)))
                   for cs in itertools.combinations(range(1, b), p - 1))
        assert max(w[c[k]:c[k + 1]].sum() for k in range(p)) <= best + 1e-12


def test_route_rows_band_mask():
    part = D.partition_pixels(64, 64, 16, 4, canon_rows=1)
    tmin = np.array([[0, 0], [1, 1], [0, 3], [2, 0]])
    tmax = np.array([[0, 0], [2, 2], [3, 3], [2, 3]])
    mask = D.route_rows(tmin, tmax, part)
    np.testing.assert_array_equal(mask, [[1, 0, 0, 0], [0, 1, 1, 0], [0, 0, 0, 1], [1, 1, 1, 1]])


def test_estimate_min_workers():
    assert D.estimate_min_workers(18_000_000, 11_200_000) == 2
    with pytest.raises(ValueError):
        D.estimate_min_workers(1, 0)


def test_reduce_gradients_fused_protocol_errors():
    smap = D.partition_gaussians(6, 2)
    chunk = D.GradChunk(0, np.array([5]), np.zeros((1, 2)), np.zeros((1, 3)), np.zeros((1, 3)),
                        np.zeros(1))
    with pytest.raises(D.ProtocolError, match="duplicate message"):
        D.reduce_gradients_fused([D.GradMessage(0, 0, []), D.GradMessage(0, 0, [])], smap)
    with pytest.raises(D.ProtocolError, match="unknown destination"):
        D.reduce_gradients_fused([D.GradMessage(0, 5, [chunk])], smap)


# --------------------------------------------------------- gloo, world 2 --

def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = D.TorchComm()
        # all-to-all-v: rank r sends (r+1)*(d+1) rows to d, rows tagged (src, dst, k)
        counts = [(rank + 1) * (d + 1) for d in range(world)]
        rows = []
        for d_ in range(world):
            for k in range(counts[d_]):
                rows.append([rank, d_, k] + [0] * 17)
        send = torch.tensor(rows, dtype=torch.int32)
        recv, rc = comm.alltoallv(send, counts)
        exp = []
        for src in range(world):
            for k in range((src + 1) * (rank + 1)):
                exp.append([src, rank, k] + [0] * 17)
        ok_a2a = torch.equal(recv, torch.tensor(exp, dtype=torch.int32)) and \
            rc == [(s + 1) * (rank + 1) for s in range(world)]
        # halo: first 2 rows to prev, last 3 rows to next
        band = torch.full((6, 4, 3), float(rank))
        to_prev = band[:2] if rank > 0 else None
        to_next = band[-3:] if rank + 1 < world else None
        gp, gn = comm.halo(to_prev, to_next, (3, 4, 3) if rank > 0 else None,
                           (2, 4, 3) if rank + 1 < world else None, torch.float32,
                           torch.device("cpu"))
        ok_halo = True
        if rank > 0:
            ok_halo &= gp.shape == (3, 4, 3) and bool((gp == rank - 1).all())
        if rank + 1 < world:
            ok_halo &= gn.shape == (2, 4, 3) and bool((gn == rank + 1).all())
        # disjoint block partials + all-reduce sum is exact
        parts = torch.zeros(8, dtype=torch.float64)
        parts[rank * 4:(rank + 1) * 4] = torch.tensor([0.1, 1e-17, -3.0, 1e300]) * (rank + 1)
        comm.allreduce_sum_(parts)
        ref = torch.cat([torch.tensor([0.1, 1e-17, -3.0, 1e300]) * (r + 1) for r in range(world)])
        ok_red = torch.equal(parts, ref)
        # per-destination counts (3 int64 per pair) and point-to-point segments
        mine = torch.tensor([[10 * rank + d, rank, d] for d in range(world)], dtype=torch.int64)
        got = torch.empty((world, world, 3), dtype=torch.int64)
        comm.counts(mine, got)
        ok_counts = torch.equal(got, torch.tensor(
            [[[10 * s + d, s, d] for d in range(world)] for s in range(world)]))
        peer = 1 - rank
        keys = torch.arange(5, dtype=torch.int64) + 100 * rank
        pay = torch.full((5, 16), rank, dtype=torch.int32)
        rk = torch.zeros(7, dtype=torch.int64)
        rp = torch.zeros((7, 16), dtype=torch.int32)
        comm.exchange([(peer, [keys, pay], [rk[1:6], rp[1:6]])])
        ok_counts &= torch.equal(rk[1:6], torch.arange(5) + 100 * peer) and \
            bool((rp[1:6] == peer).all()) and int(rk[0]) == 0 and int(rk[6]) == 0
        q.put((rank, ok_a2a and ok_counts, ok_halo, ok_red))
    finally:
        dist.destroy_process_group()


def test_collectives_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, a2a, halo, red in results:
        assert a2a, f"rank {rank} all-to-all-v"
        assert halo, f"rank {rank} halo"
        assert red, f"rank {rank} all-reduce"


# ------------------------------------------- densify exchange, gloo world 2 --

def _densify_inputs():
    """Densify fixture cloud (reference make_golden.py --densify) with seeded
    Adam moments; thresholds from the fixture."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from golden_io import cloud_from, load
    from paper_2509_05216_b200.gaussians import PARAM_NAMES, GaussianCloud
    d = load("densify")
    src = cloud_from(d, "in_")
    cloud = GaussianCloud(*(torch.from_numpy(np.ascontiguousarray(getattr(src, k)))
                            for k in PARAM_NAMES), degree=int(src.degree))
    g = torch.Generator().manual_seed(5)
    m = {k: torch.randn(getattr(cloud, k).shape, generator=g) for k in PARAM_NAMES}
    v = {k: torch.rand(getattr(cloud, k).shape, generator=g) for k in PARAM_NAMES}
    return d, cloud, m, v


def _densify_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from types import SimpleNamespace
        import paper_2509_05216_b200 as P
        from paper_2509_05216_b200.gaussians import PARAM_NAMES, GaussianCloud
        d, cloud, m, v = _densify_inputs()
        smap = D.partition_gaussians(cloud.count, world)
        a, b = smap.starts[rank], smap.starts[rank + 1]
        rs = SimpleNamespace(
            cloud=GaussianCloud(*(getattr(cloud, k)[a:b].clone() for k in PARAM_NAMES),
                                degree=cloud.degree),
            m={k: m[k][a:b].clone() for k in PARAM_NAMES},
            v={k: v[k][a:b].clone() for k in PARAM_NAMES},
            seen=torch.from_numpy(d["seen"][a:b].copy()),
            grad_accum=torch.from_numpy(d["grad_accum"][a:b].copy()),
            cfg=P.TrainConfig(seed=int(d["seed"])), id_base=a, n=b - a)
        rows, new_map = D.densify_exchange(rs, D.TorchComm(), int(d["iteration"]),
                                           float(d["grad_thr"]), float(d["split_thr"]))
        params, mm, vv = D.unpack_rows(rows, cloud.degree)
        q.put((rank, {k: params[k].numpy() for k in PARAM_NAMES},
               {k: mm[k].numpy() for k in PARAM_NAMES}, {k: vv[k].numpy() for k in PARAM_NAMES},
               new_map.starts))
    finally:
        dist.destroy_process_group()


def test_densify_exchange_world2_gloo_equals_single():
    """Sharded densify (local classify, global id reassignment, all-to-all-v to
    the rebalanced contiguous shards) == one worker's densify, bit for bit."""
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200.densify import carry_moments
    from paper_2509_05216_b200.gaussians import PARAM_NAMES
    from paper_2509_05216_b200.training import TrainStats
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_densify_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = sorted([q.get(timeout=180) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    d, cloud, m, v = _densify_inputs()
    stats = TrainStats(grad_accum=torch.from_numpy(d["grad_accum"]),
                       seen=torch.from_numpy(d["seen"]))
    new, mapping = P.densify_and_prune(cloud, stats, P.TrainConfig(seed=int(d["seed"])),
                                       int(d["iteration"]), float(d["grad_thr"]),
                                       float(d["split_thr"]))
    m1, v1 = carry_moments(m, mapping, new), carry_moments(v, mapping, new)
    starts = results[0][4]
    assert starts[-1] == new.count and results[1][4] == starts
    for rank, params, mm, vv, _ in results:
        a, b = starts[rank], starts[rank + 1]
        for k in PARAM_NAMES:
            assert np.array_equal(params[k], getattr(new, k)[a:b].numpy()), (rank, k)
            assert np.array_equal(mm[k], m1[k][a:b].numpy()), (rank, "m", k)
            assert np.array_equal(vv[k], v1[k][a:b].numpy()), (rank, "v", k)


# ------------------------------------- reference data-plane helpers (fixtures) --

def _dataplane():
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from golden_io import load
    return load("dataplane")


def test_rebalance_matches_reference():
    """rebalance(shard_map, counts) == the reference's plan and resulting map
    (distributed.py:229-268; tests/golden/make_golden_dist.py)."""
    d = _dataplane()
    for case in range(6):
        owner = d[f"rb{case}_owner"]
        w = int(owner.max()) + 1
        smap = D.ShardMap.from_lists([np.nonzero(owner == k)[0] for k in range(w)], int(d[f"rb{case}_n"]))
        plan, new = D.rebalance(smap, smap.sizes)
        assert np.array_equal(np.array(plan, dtype=np.int64).reshape(-1, 3), d[f"rb{case}_plan"])
        assert np.array_equal(new.owner, d[f"rb{case}_new_owner"])
        sizes = new.sizes
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        D.rebalance(smap, [1] * smap.workers)


def test_route_splats_matches_reference():
    """route_splats over the reference's round-robin tile assignment."""
    from types import SimpleNamespace
    from paper_2509_05216_b200.rasterizer import ProjectedSplat
    d = _dataplane()
    spl = [ProjectedSplat(gaussian_index=int(i), mean2d=np.zeros(2), cov2d=np.zeros(3),
                          depth=float(z), color=np.zeros(3), opacity=0.5,
                          tile_span=((int(s[0]), int(s[1])), (int(s[2]), int(s[3]))))
           for s, z, i in zip(d["rs_spans"], d["rs_depth"], d["rs_index"])]
    part = SimpleNamespace(workers=3, tiles_x=7, assignment=d["rs_assignment"])
    lists = D.route_splats(spl, part)
    for w in range(3):
        assert [s.gaussian_index for s in lists[w]] == d[f"rs_list{w}"].tolist()
    # row bands: a splat reaches exactly the bands its rows overlap
    bands = D.partition_pixels(7 * 16, 8 * 16, 16, 2, canon_rows=2)
    lists = D.route_splats(spl, bands)
    for s in spl:
        (_, y0), (_, y1) = s.tile_span
        want = [w for w in range(2) if y0 < bands.band_rows[w + 1] and y1 >= bands.band_rows[w]]
        got = [w for w in range(2) if any(t is s for t in lists[w])]
        assert got == want


def test_exchange_layout_places_every_segment_once():
    """The peer-store exchange writes each shard's records straight into the
    destination band's buffer at exchange_layout(...)["pack_at"], and each
    band's block records into the owner's buffer at ["grad_at"]: those must be
    exactly the segment starts the receiving side reads (source order for
    splat records, band order for gradient records), every rank computing
    them from the same all-gathered matrix, and the capacities must cover
    every rank's receive totals."""
    rng = np.random.default_rng(5)
    for W in (1, 2, 3, 8):
        mat = rng.integers(0, 50, size=(W, W, 3)).astype(np.int64)
        mat[rng.random((W, W)) < 0.3] = 0
        lays = [D.exchange_layout(mat, r) for r in range(W)]
        for d in range(W):
            recv = mat[:, d, 0]
            starts = np.concatenate([[0], np.cumsum(recv)])
            for s_ in range(W):
                assert lays[s_]["pack_at"][d] == starts[s_]
            assert starts[-1] <= lays[d]["need_r"]
        for s_ in range(W):
            # owner s receives band b's records at grad_seg[b]; band b writes at grad_at[s]
            for b in range(W):
                assert lays[b]["grad_at"][s_] == lays[s_]["grad_seg"][b]
            assert lays[s_]["grad_seg"][-1] == mat[s_, :, 1].sum() <= lays[s_]["need_g"]
        assert len({(l["need_r"], l["need_g"]) for l in lays}) == 1
