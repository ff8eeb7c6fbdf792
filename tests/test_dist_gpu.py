"""Bitwise GPU-count invariance of the sharded step, on one B200.

The multi-GPU step (paper_2509_05216_b200/distributed.py) is a sequence of
per-rank phases separated by collectives.  Here W ranks' phases run in
sequence on ONE GPU with the collectives replaced by in-process copies (no
kernel ever waits on another rank), which exercises every data-plane kernel
(route, pack/unpack, band binning, halo'd loss, per-block fold, owner fold)
and must reproduce the single-GPU engine bit for bit -- the reference's
headline property (tests/test_acceptance.py:101-123 of the reference)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from golden_io import cam_from, load

pytestmark = pytest.mark.gpu


def _setup():
    import paper_2509_05216_b200 as P
    d = load("config1")
    cams = []
    for i in range(d["images_u8"].shape[0]):
        c = cam_from(d, prefix=f"cam{i}_")
        cams.append(P.Camera(c.rotation, c.translation, c.fx, c.fy, c.cx, c.cy, c.width, c.height))
    gt = torch.from_numpy(d["images_u8"]).cuda()
    cloud = P.cloud_from_points(d["points"], d["init_log_scales"])
    return P, d, cams, gt, cloud


def _run_single(P, cams, gt, cloud, iters, canon):
    from paper_2509_05216_b200.engine import Trainer
    cfg = P.TrainConfig(iterations=iters, densify=False)
    tr = Trainer(cloud.copy(), cams[0].width, cams[0].height, cfg, _extent(cams), canon_rows=canon)
    sched = P.build_schedule(iters, len(cams), 0)
    for it in range(1, iters + 1):
        tr.step(it, cams[sched[it - 1]], gt[sched[it - 1]])
    torch.cuda.synchronize()
    return tr.loss_dev[1:iters + 1].tolist(), tr.cloud


def _run_emulated(P, cams, gt, cloud, iters, canon, workers, total=None, peers=False):
    from paper_2509_05216_b200 import distributed as D
    cfg = P.TrainConfig(iterations=total or iters, densify=False)
    ranks, smap, part = D.make_ranks(cloud.copy(), cams[0].width, cams[0].height, cfg, _extent(cams),
                                     workers, torch.device("cuda", 0), canon_rows=canon)
    sched = P.build_schedule(total or iters, len(cams), 0)
    losses = []
    for it in range(1, iters + 1):
        loss = D.emulated_step(ranks, cams[sched[it - 1]], gt[sched[it - 1]], it, peers=peers)
        losses.append(float(loss[0]))
    torch.cuda.synchronize()
    return losses, D.gather_cloud(ranks), part


@pytest.mark.parametrize("peers", [False, True], ids=["p2p_copies", "peer_stores"])
@pytest.mark.parametrize("workers", [1, 2, 3, 4])
def test_sharded_step_bitwise_equals_single_gpu(workers, peers):
    """peer_stores: the pack, forward-halo and band-fold kernels write straight
    into the other ranks' buffers (the peer-store exchange's layout)."""
    P, d, cams, gt, cloud = _setup()
    iters, canon = 4, 1
    ref_losses, ref_cloud = _run_single(P, cams, gt, cloud, iters, canon)
    losses, got, part = _run_emulated(P, cams, gt, cloud, iters, canon, workers, peers=peers)
    assert len(part.band_rows) == workers + 1
    assert losses == ref_losses, (losses, ref_losses)
    for k in P.PARAM_NAMES:
        assert torch.equal(getattr(got, k), getattr(ref_cloud, k)), k


def test_sharded_losses_track_reference():
    """The W=2 sharded run also tracks the reference's own loss trajectory."""
    P, d, cams, gt, cloud = _setup()
    losses, _, _ = _run_emulated(P, cams, gt, cloud, 10, 1, 2, total=100)
    ref = np.array(d["losses"][:10])
    assert np.max(np.abs(np.array(losses) - ref) / ref) <= 2e-3


def _extent(cams):
    from oracle import train as T
    return T.scene_extent(cams)


def _run_single_densify(P, cams, gt, cloud, iters, canon, cfg):
    from paper_2509_05216_b200.engine import Trainer
    tr = Trainer(cloud.copy(), cams[0].width, cams[0].height, cfg, _extent(cams), canon_rows=canon)
    sched = P.build_schedule(iters, len(cams), 0)
    for it in range(1, iters + 1):
        tr.step(it, cams[sched[it - 1]], gt[sched[it - 1]])
        if tr.densify_due(it):
            tr.densify(it)
    torch.cuda.synchronize()
    return tr.loss_dev[1:iters + 1].tolist(), tr.cloud


@pytest.mark.parametrize("peers", [False, True], ids=["p2p_copies", "peer_stores"])
@pytest.mark.parametrize("workers", [2, 3])
def test_sharded_densify_bitwise_equals_single_gpu(workers, peers):
    """Densify + rebalance inside the sharded engine (emulated ranks) keeps
    the run bitwise equal to the single-GPU engine across the event."""
    from paper_2509_05216_b200 import distributed as D
    P, d, cams, gt, cloud = _setup()
    iters, canon = 5, 1
    cfg = P.TrainConfig(iterations=iters, densify_start=2, densify_interval=2, densify_stop=4)
    ref_losses, ref_cloud = _run_single_densify(P, cams, gt, cloud, iters, canon, cfg)
    assert ref_cloud.count != cloud.count
    ranks, smap, part = D.make_ranks(cloud.copy(), cams[0].width, cams[0].height, cfg,
                                     _extent(cams), workers, torch.device("cuda", 0),
                                     canon_rows=canon)
    sched = P.build_schedule(iters, len(cams), 0)
    losses = []
    for it in range(1, iters + 1):
        loss = D.emulated_step(ranks, cams[sched[it - 1]], gt[sched[it - 1]], it, peers=peers)
        losses.append(float(loss[0]))
        if D.densify_due(cfg, it):
            ranks = D.emulated_densify(ranks, it)
    got = D.gather_cloud(ranks)
    assert losses == ref_losses, (losses, ref_losses)
    for k in P.PARAM_NAMES:
        assert torch.equal(getattr(got, k), getattr(ref_cloud, k)), k


@pytest.mark.parametrize("peers", [False, True], ids=["p2p_copies", "peer_stores"])
def test_sharded_step_with_nothing_visible(peers):
    """A view that sees no Gaussian (camera turned 180 degrees about its y
    axis) between ordinary ones: every rank routes, packs and renders nothing,
    and the W=3 run stays bitwise the single-GPU run."""
    from paper_2509_05216_b200 import distributed as D
    from paper_2509_05216_b200.engine import Trainer
    P, d, cams, gt, cloud = _setup()
    iters, canon = 4, 1
    sched = P.build_schedule(iters, len(cams), 0)
    c0 = cams[sched[1]]
    flip = np.diag([-1.0, 1.0, -1.0])
    away = P.Camera(flip @ np.asarray(c0.rotation), flip @ np.asarray(c0.translation),
                    c0.fx, c0.fy, c0.cx, c0.cy, c0.width, c0.height)
    views = [cams[sched[0]], away, cams[sched[2]], away]
    cfg = P.TrainConfig(iterations=iters, densify=False)
    tr = Trainer(cloud.copy(), c0.width, c0.height, cfg, _extent(cams), canon_rows=canon)
    for it in range(1, iters + 1):
        tr.step(it, views[it - 1], gt[sched[it - 1]])
    torch.cuda.synchronize()
    ref_losses = tr.loss_dev[1:iters + 1].tolist()
    ranks, smap, part = D.make_ranks(cloud.copy(), c0.width, c0.height, cfg, _extent(cams), 3,
                                     torch.device("cuda", 0), canon_rows=canon)
    losses = [float(D.emulated_step(ranks, views[it - 1], gt[sched[it - 1]], it, peers=peers)[0])
              for it in range(1, iters + 1)]
    got = D.gather_cloud(ranks)
    assert losses == ref_losses, (losses, ref_losses)
    for k in P.PARAM_NAMES:
        assert torch.equal(getattr(got, k), getattr(tr.cloud, k)), k


@pytest.mark.parametrize("peers", [False, True], ids=["p2p_copies", "peer_stores"])
@pytest.mark.parametrize("wh", [(70, 45), (33, 97)])
def test_sharded_ragged_image_bitwise_equals_single_gpu(wh, peers):
    """Image sizes with partial edge tiles (bands end inside a tile row's
    pixels at the bottom; the last tile column is partial): W=3 emulated ranks
    == one GPU, bit for bit, over 4 iterations."""
    from paper_2509_05216_b200 import distributed as D
    from paper_2509_05216_b200.engine import Trainer
    P, d, cams, gt, cloud = _setup()
    W, H = wh
    iters, canon = 4, 1
    cams = [P.Camera(c.rotation, c.translation, c.fx * W / c.width, c.fx * W / c.width,
                     0.5 * W, 0.5 * H, W, H) for c in cams]
    rng = np.random.default_rng(5)
    gt = torch.from_numpy(rng.integers(0, 256, (len(cams), H, W, 3), dtype=np.uint8)).cuda()
    ref_losses, ref_cloud = _run_single(P, cams, gt, cloud, iters, canon)
    losses, got, part = _run_emulated(P, cams, gt, cloud, iters, canon, 3, peers=peers)
    assert losses == ref_losses, (losses, ref_losses)
    for k in P.PARAM_NAMES:
        assert torch.equal(getattr(got, k), getattr(ref_cloud, k)), k


@pytest.mark.parametrize("peers", [False, True], ids=["p2p_copies", "peer_stores"])
def test_sharded_two_entry_backward_bitwise_equals_single_gpu(peers):
    """Band launches small enough for the several-entries-per-step backward
    (engine.UNROLL2_TILES) while the single-GPU launch walks one entry per
    step: the W=2 run is still bitwise the single-GPU run."""
    from paper_2509_05216_b200 import engine as E
    P, d, cams, gt, cloud = _setup()
    iters, canon = 4, 1
    saved = E.UNROLL2_TILES, E.CHUNK
    try:
        E.UNROLL2_TILES, E.CHUNK = 15, 0  # 16 tiles on one GPU, fewer per band at W = 2
        ref_losses, ref_cloud = _run_single(P, cams, gt, cloud, iters, canon)
        losses, got, part = _run_emulated(P, cams, gt, cloud, iters, canon, 2, peers=peers)
    finally:
        E.UNROLL2_TILES, E.CHUNK = saved
    assert losses == ref_losses, (losses, ref_losses)
    for k in P.PARAM_NAMES:
        assert torch.equal(getattr(got, k), getattr(ref_cloud, k)), k


@pytest.mark.parametrize("peers", [False, True], ids=["p2p_copies", "peer_stores"])
def test_sharded_chunked_multi_entry_backward_bitwise_equals_single_gpu(peers):
    """Chunked backward (config 1 chunks its lists) with the several-entries-
    per-step instantiation in the W=2 bands only: still bitwise one GPU."""
    from paper_2509_05216_b200 import engine as E
    P, d, cams, gt, cloud = _setup()
    iters, canon = 4, 1
    saved = E.UNROLL2_TILES
    try:
        E.UNROLL2_TILES = 15  # 16 tiles on one GPU, fewer per band at W = 2
        ref_losses, ref_cloud = _run_single(P, cams, gt, cloud, iters, canon)
        losses, got, part = _run_emulated(P, cams, gt, cloud, iters, canon, 2, peers=peers)
    finally:
        E.UNROLL2_TILES = saved
    assert losses == ref_losses, (losses, ref_losses)
    for k in P.PARAM_NAMES:
        assert torch.equal(getattr(got, k), getattr(ref_cloud, k)), k
