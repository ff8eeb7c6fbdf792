"""End-to-end training parity on the GPU: the device-resident engine against
the reference's own training runs (tests/golden/train_tiny.npz and
config1.npz: BASELINE config 1, sphere 20K G, 64^2, 16 views, 100 its).

Bars: per-iteration loss rel. err <= 2e-4 (float32 raster vs the reference's
float64); final PSNR within 0.05 dB and SSIM within 2e-3 of the reference;
two runs bitwise identical (deterministic reductions everywhere)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from golden_io import cam_from, load

pytestmark = pytest.mark.gpu


def _dataset(d, key_images, count):
    import paper_2509_05216_b200 as P
    cams = []
    for i in range(count):
        c = cam_from(d, prefix=f"cam{i}_")
        cams.append(P.Camera(c.rotation, c.translation, c.fx, c.fy, c.cx, c.cy, c.width, c.height))
    imgs = d[key_images]
    if imgs.dtype == np.uint8:
        imgs = (imgs.astype(np.float64) / 255.0).astype(np.float32)
    pts = P.PointCloud(d["points"], d["normals"])
    return P.TrainDataset(cameras=cams, images=imgs, points=pts)


def _init(d, prefix=None):
    import paper_2509_05216_b200 as P
    if prefix:
        from golden_io import cloud_from
        return cloud_from(d, prefix)
    return P.cloud_from_points(d["points"], d["init_log_scales"])


def test_train_tiny_matches_reference():
    import paper_2509_05216_b200 as P
    d = load("train_tiny")
    ds = _dataset(d, "images", d["images"].shape[0])
    cfg = P.TrainConfig(iterations=6, eval_interval=3, densify=False, seed=4)
    cloud, rep = P.train_single(ds, cfg, init_cloud=_init(d, "init_"))
    ref = np.array(d["losses"])
    got = np.array(rep.iteration_losses)
    assert np.max(np.abs(got - ref) / ref) <= 2e-4, (got, ref)
    assert [r.iteration for r in rep.records] == list(d["rec_iter"])
    for r, p, s in zip(rep.records, d["rec_psnr"], d["rec_ssim"]):
        assert abs(r.psnr - p) <= 0.05 and abs(r.ssim - s) <= 2e-3
    for k in P.PARAM_NAMES:
        a = getattr(cloud, k).cpu().numpy()
        b = d["final_" + k]
        assert np.abs(a - b).max() <= 1e-3 * max(1.0, np.abs(b).max()), k


def test_config1_psnr_parity_and_determinism():
    import paper_2509_05216_b200 as P
    d = load("config1")
    ds = _dataset(d, "images_u8", d["images_u8"].shape[0])
    cfg = P.TrainConfig(iterations=100, eval_interval=0, seed=0)
    _, rep = P.train_single(ds, cfg, init_cloud=_init(d))
    assert abs(rep.records[0].psnr - float(d["rec_psnr"][0])) <= 0.01
    assert abs(rep.final.psnr - float(d["rec_psnr"][-1])) <= 0.05, (rep.final.psnr, d["rec_psnr"])
    assert abs(rep.final.ssim - float(d["rec_ssim"][-1])) <= 2e-3
    ref = np.array(d["losses"])
    got = np.array(rep.iteration_losses)
    assert np.max(np.abs(got - ref) / ref) <= 2e-3
    _, rep2 = P.train_single(ds, cfg, init_cloud=_init(d), evaluate=False)
    assert rep2.iteration_losses == rep.iteration_losses


def test_resume_from_train_state_is_bitwise(tmp_path):
    """save_train_state / load_train_state (SSGC cloud + Adam moments + stats)
    resume a run bit for bit."""
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200.engine import Trainer
    d = load("train_tiny")
    ds = _dataset(d, "images", d["images"].shape[0])
    cfg = P.TrainConfig(iterations=6, densify=False, seed=4)
    gt = torch.from_numpy(np.ascontiguousarray(d["images"])).cuda()
    sched = P.build_schedule(6, ds.view_count, 4)

    def fresh():
        return Trainer(P.to_device_cloud(_init(d, "init_")), ds.width, ds.height, cfg,
                       ds.scene_extent)

    a = fresh()
    for it in range(1, 7):
        a.step(it, ds.cameras[sched[it - 1]], gt[sched[it - 1]])
    b = fresh()
    for it in range(1, 4):
        b.step(it, ds.cameras[sched[it - 1]], gt[sched[it - 1]])
    path = str(tmp_path / "run.ssgc")
    P.save_train_state(path, b, 3)
    c = fresh()
    start = P.load_train_state(path, c)
    assert start == 3
    for it in range(start + 1, 7):
        c.step(it, ds.cameras[sched[it - 1]], gt[sched[it - 1]])
    for k in P.PARAM_NAMES:
        assert torch.equal(getattr(a.cloud, k), getattr(c.cloud, k)), k


def test_contribution_masks_change_no_result():
    """The training lists and raster pair (isg_bin_emit_live: pairs no pixel of
    their tile can composite have no entry and no subtotal slot;
    isg_raster_fwd_masked / isg_raster_bwd_masked: the backward walks only the
    entries the forward composited; isg_reduce_live folds the live slots) ==
    the full lists and the unmasked pair: images and T_final bitwise, 2-D
    gradients equal (== ignores the sign of zero), and the parameters after 4
    training iterations bitwise."""
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200.engine import Trainer
    d = load("config1")
    ds = _dataset(d, "images_u8", d["images_u8"].shape[0])
    cfg = P.TrainConfig(iterations=4, densify=False, seed=0)
    gt = _images(ds)
    sched = P.build_schedule(4, ds.view_count, 0)
    runs = []
    for masked in (True, False):
        t = Trainer(P.to_device_cloud(_init(d)), ds.width, ds.height, cfg, ds.scene_extent)
        t.r.use_cmask = masked
        t.r.chunk = 0  # one backward CTA per tile: the same arithmetic as the unmasked pair
        t.r.keep_grad2d = True
        for it in range(1, 5):
            t.step(it, ds.cameras[sched[it - 1]], gt[sched[it - 1]])
        torch.cuda.synchronize()
        runs.append(t)
    a, b = runs
    assert a.r.cmask_ok and not b.r.cmask_ok
    assert torch.equal(a.r.image, b.r.image) and torch.equal(a.r.t_final, b.r.t_final)
    # (n_last are list positions: the culled lists are shorter)
    assert a.r.live and int(a.r.offsets[-1]) < int(b.r.offsets[-1])
    assert torch.equal(a.r.grad2d, b.r.grad2d)
    for k in P.PARAM_NAMES:
        assert torch.equal(getattr(a.cloud, k), getattr(b.cloud, k)), k


def test_backward_chunking_matches_one_cta_per_tile():
    """The chunked backward (isg_chunks: long lists cut into 32-entry-aligned
    chunks, each started from the forward's boundary state) against one CTA
    per tile: images bitwise (the forward only records state), 2-D gradients
    within float32 rounding of the chunk-start colour (S = image - C), and
    4 training iterations within the same bar."""
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200.engine import Trainer
    d = load("config1")
    ds = _dataset(d, "images_u8", d["images_u8"].shape[0])
    cfg = P.TrainConfig(iterations=4, densify=False, seed=0)
    gt = _images(ds)
    sched = P.build_schedule(4, ds.view_count, 0)
    runs = []
    for chunk in (64, 0):  # config 1 lists reach 6.3K entries: many chunks per tile
        t = Trainer(P.to_device_cloud(_init(d)), ds.width, ds.height, cfg, ds.scene_extent)
        t.r.chunk = chunk
        t.r.keep_grad2d = True
        for it in range(1, 5):
            t.step(it, ds.cameras[sched[it - 1]], gt[sched[it - 1]])
            if it == 1:
                g1 = t.r.grad2d.clone()
                img1 = t.r.image.clone()
        torch.cuda.synchronize()
        runs.append((t, g1, img1))
    (a, ga, ia), (b, gb, ib) = runs
    assert a.r.chunks is not None and a.r.chunks.chunk == 64
    assert b.r.chunks is None or b.r.chunks.chunk == 0  # (unchunked; maybe two entries per step)
    assert torch.equal(ia, ib)
    rel = float((ga - gb).abs().max() / gb.abs().max())
    assert rel <= 1e-4, rel
    la, lb = a.loss_dev[1:5], b.loss_dev[1:5]
    assert float(((la - lb).abs() / lb).max()) <= 1e-6
    for k in P.PARAM_NAMES:
        x, y = getattr(a.cloud, k), getattr(b.cloud, k)
        assert float((x - y).abs().max()) <= 2.5 * 4 * 5e-2, k  # Adam's bound (lr_opacity)


def _images(ds):
    imgs = torch.from_numpy(np.ascontiguousarray(ds.images)).cuda()
    if imgs.dtype == torch.uint8:
        imgs = (imgs.to(torch.float64) / 255.0).to(torch.float32)
    return imgs


def test_culled_lists_are_ordered_sublists_of_the_full_lists():
    """isg_bin_emit_live keeps, per tile, a subsequence of the reference's
    list (same relative order); every live slot appears in exactly one list,
    and its subtotal record carries its tile row (the fold's block key)."""
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200.engine import Trainer
    d = load("config1")
    ds = _dataset(d, "images_u8", d["images_u8"].shape[0])
    cfg = P.TrainConfig(iterations=1, densify=False, seed=0)
    lists = []
    for masked in (True, False):
        t = Trainer(P.to_device_cloud(_init(d)), ds.width, ds.height, cfg, ds.scene_extent)
        t.r.use_cmask = masked
        ctx = t.r.forward(t.cloud, ds.cameras[0])
        torch.cuda.synchronize()
        off = t.r.offsets.cpu().numpy()
        ent = t.r.entries[:int(off[-1])].cpu().numpy()
        if masked:
            slots = ent.copy()
            ent = t.r.slot_rank[:ctx.e].cpu().numpy()[ent]  # slots -> ranks
            live_slots = ctx.e
            off_live = off
            tr = t
        lists.append([ent[off[k]:off[k + 1]] for k in range(len(off) - 1)])
    culled_total = 0
    for lc, lf in zip(*lists):
        assert np.all(np.isin(lc, lf))
        pos = np.searchsorted(lf, lc)  # both lists ascend in rank
        assert np.array_equal(lf[pos], lc) and np.all(np.diff(pos) > 0)
        culled_total += len(lf) - len(lc)
    assert culled_total > 0
    assert np.array_equal(np.sort(slots), np.arange(live_slots))
    # the backward's records: tile row of every slot in float 9
    tr.step(1, ds.cameras[0], _images(ds)[0])
    torch.cuda.synchronize()
    rows = tr.r.partials[:live_slots, 9].contiguous().view(torch.int32).cpu().numpy()
    tiles_x = tr.r.tiles_x
    tile_of = np.repeat(np.arange(len(off_live) - 1), np.diff(off_live))
    want = np.empty(live_slots, dtype=np.int64)
    want[slots] = tile_of // tiles_x
    assert np.array_equal(rows, want)


@pytest.mark.parametrize("densify", [False, True])
def test_fused_chain_adam_is_bitwise_the_separate_launches(densify):
    """isg_chain_fold_adam (fold + chain + stats + Adam in one pass, gradients
    kept in registers) == isg_chain_fold_train + isg_adam_groups: parameters,
    moments and statistics bitwise after 6 iterations (with a densify event,
    which reads the statistics)."""
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200 import engine as E
    from paper_2509_05216_b200.engine import Trainer
    d = load("config1")
    ds = _dataset(d, "images_u8", d["images_u8"].shape[0])
    cfg = P.TrainConfig(iterations=6, densify=densify, densify_start=2, densify_interval=2,
                        densify_stop=5, seed=0)
    gt = _images(ds)
    sched = P.build_schedule(6, ds.view_count, 0)
    runs = []
    saved = E.FUSE_ADAM
    try:
        for fused in (True, False):
            E.FUSE_ADAM = fused
            t = Trainer(P.to_device_cloud(_init(d)), ds.width, ds.height, cfg, ds.scene_extent)
            for it in range(1, 7):
                t.step(it, ds.cameras[sched[it - 1]], gt[sched[it - 1]])
                if t.densify_due(it):
                    t.densify(it)
            torch.cuda.synchronize()
            runs.append(t)
    finally:
        E.FUSE_ADAM = saved
    a, b = runs
    assert torch.equal(a.loss_dev, b.loss_dev)
    for k in P.PARAM_NAMES:
        assert torch.equal(getattr(a.cloud, k), getattr(b.cloud, k)), k
        assert torch.equal(a.m[k], b.m[k]) and torch.equal(a.v[k], b.v[k]), k
    assert torch.equal(a.stats.seen, b.stats.seen)
    assert torch.equal(a.stats.grad_accum, b.stats.grad_accum)


def test_training_step_beyond_65536_tiles():
    """An 8192^2 image (262144 tiles): 4-byte tile keys through the live
    emission, the tile sort, the offsets and the bucketed launch order; three
    training steps run with finite losses."""
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200 import synthetic as S
    from paper_2509_05216_b200.engine import Trainer
    from paper_2509_05216_b200.training import TrainConfig, TrainDataset, PointCloud, build_schedule
    dev = torch.device("cuda", 0)
    res = 8192
    nv = S.CONFIGS["config2"][4]
    sched = build_schedule(3, nv, 0)
    wl = S.make_workload("config2", dev, view_ids=sched, resolution=res)
    ext = TrainDataset(wl.cameras, np.zeros((nv, 1, 1, 3)),
                       PointCloud(wl.points, wl.normals)).scene_extent
    tr = Trainer(P.cloud_from_points(wl.points, wl.log_scales, 1, dev), res, res,
                 TrainConfig(iterations=3, densify=False), ext, dev)
    for it in range(1, 4):
        tr.step(it, wl.cameras[sched[it - 1]], wl.images_u8[it - 1])
    torch.cuda.synchronize()
    assert tr.r.n_tiles == 262144 and tr.r.live
    losses = tr.loss_dev[1:4].cpu().numpy()
    assert np.isfinite(losses).all() and (losses > 0).all()
    off = tr.r.offsets.cpu().numpy()
    assert off[0] == 0 and (np.diff(off) >= 0).all() and off[-1] > 0


def test_launch_order_changes_no_result():
    """The raster pair's launch order (heaviest lists first: the one-launch
    bucketed order, the exact 16-bit sort, or plain list order) is the launch
    order only: losses and parameters after 4 iterations are bitwise equal."""
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200 import engine as E
    from paper_2509_05216_b200.engine import Trainer
    d = load("config1")
    ds = _dataset(d, "images_u8", d["images_u8"].shape[0])
    cfg = P.TrainConfig(iterations=4, densify=False, seed=0)
    gt = _images(ds)
    sched = P.build_schedule(4, ds.view_count, 0)
    saved = E.EXACT_ORDER
    runs = []
    try:
        for heavy, exact in ((True, False), (True, True), (False, False)):
            E.EXACT_ORDER = exact
            t = Trainer(P.to_device_cloud(_init(d)), ds.width, ds.height, cfg, ds.scene_extent)
            t.r.heavy_first = heavy
            for it in range(1, 5):
                t.step(it, ds.cameras[sched[it - 1]], gt[sched[it - 1]])
            torch.cuda.synchronize()
            order = t.r.tile_order.clone() if t.r.tile_order is not None else None
            runs.append((t, order))
    finally:
        E.EXACT_ORDER = saved
    (a, oa), (b, ob), (c, oc) = runs
    n = a.r.n_tiles
    assert oc is None and sorted(oa[:n].tolist()) == list(range(n))
    assert sorted(ob[:n].tolist()) == list(range(n))
    for t in (b, c):
        assert torch.equal(a.loss_dev, t.loss_dev)
        for k in P.PARAM_NAMES:
            assert torch.equal(getattr(a.cloud, k), getattr(t.cloud, k)), k


def test_graph_captured_presync_equals_eager():
    """The pre-sync launches as a CUDA graph replay (camera uploaded to device
    memory, re-captured when densify replaces the cloud) == eager launches:
    losses, parameters and statistics bitwise over 6 iterations."""
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200 import engine as E
    from paper_2509_05216_b200.engine import Trainer
    d = load("config1")
    ds = _dataset(d, "images_u8", d["images_u8"].shape[0])
    cfg = P.TrainConfig(iterations=6, densify_start=2, densify_interval=2, densify_stop=5, seed=0)
    gt = _images(ds)
    sched = P.build_schedule(6, ds.view_count, 0)
    saved = E.GRAPH
    runs = []
    try:
        for graph in (True, False):
            E.GRAPH = graph
            t = Trainer(P.to_device_cloud(_init(d)), ds.width, ds.height, cfg, ds.scene_extent)
            for it in range(1, 7):
                t.step(it, ds.cameras[sched[it - 1]], gt[sched[it - 1]])
                if t.densify_due(it):
                    t.densify(it)
            torch.cuda.synchronize()
            runs.append(t)
    finally:
        E.GRAPH = saved
    a, b = runs
    assert a.r.graph is not None and b.r.graph is None
    assert torch.equal(a.loss_dev, b.loss_dev)
    for k in P.PARAM_NAMES:
        assert torch.equal(getattr(a.cloud, k), getattr(b.cloud, k)), k
    assert torch.equal(a.stats.seen, b.stats.seen)


def test_step_on_a_view_with_nothing_visible():
    """A view that sees no Gaussian (the camera turned 180 degrees about its y
    axis) between two ordinary ones: zero visible splats, zero entries and zero
    live slots through the graph-captured binning, the sort, the raster pair
    and the fold.  The image is the background, no statistics move, and the
    run is bitwise the same with eager pre-sync launches."""
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200 import engine as E
    from paper_2509_05216_b200.engine import Trainer
    d = load("config1")
    ds = _dataset(d, "images_u8", d["images_u8"].shape[0])
    cfg = P.TrainConfig(iterations=4, densify=False, seed=0)
    gt = _images(ds)
    sched = P.build_schedule(4, ds.view_count, 0)
    c0 = ds.cameras[sched[1]]
    flip = np.diag([-1.0, 1.0, -1.0])
    away = P.Camera(flip @ np.asarray(c0.rotation), flip @ np.asarray(c0.translation),
                    c0.fx, c0.fy, c0.cx, c0.cy, c0.width, c0.height)
    views = [ds.cameras[sched[0]], away, ds.cameras[sched[2]], away]
    saved = E.GRAPH
    runs = []
    try:
        for graph in (True, False):
            E.GRAPH = graph
            t = Trainer(P.to_device_cloud(_init(d)), ds.width, ds.height, cfg, ds.scene_extent)
            seen = []
            for it in range(1, 5):
                t.step(it, views[it - 1], gt[sched[it - 1]])
                torch.cuda.synchronize()
                seen.append(t.stats.seen.clone())
                if it == 2:
                    img = t.r.image.float().cpu().numpy()
                    assert (img == 1.0).all()  # background (1, 1, 1)
            runs.append((t, seen))
    finally:
        E.GRAPH = saved
    (a, sa), (b, sb) = runs
    assert torch.equal(sa[1], sa[0]) and torch.equal(sa[3], sa[2])
    assert int(sa[0].sum()) > 0
    losses = a.loss_dev[1:5].cpu().numpy()
    assert np.isfinite(losses).all()
    assert torch.equal(a.loss_dev, b.loss_dev)
    for k in P.PARAM_NAMES:
        assert torch.equal(getattr(a.cloud, k), getattr(b.cloud, k)), k


@pytest.mark.parametrize("wh", [(70, 45), (33, 97)])
def test_ragged_image_step_matches_oracle(wh):
    """Image sizes that are not multiples of the 16-pixel tile (partial tiles on
    the right and bottom edges): two training iterations against the oracle's
    iteration (src/engine.py:481-537) from the same pre-step state -- loss rel
    <= 2e-5, 2-D and parameter gradients within the scale-parity bars, and the
    post-step parameters bitwise the reference's Adam on the GPU's gradients."""
    import paper_2509_05216_b200 as P
    from oracle import oracle as O
    from oracle import train as T
    from paper_2509_05216_b200.engine import Trainer
    O.build()
    W, H = wh
    d = load("config1")
    ds = _dataset(d, "images_u8", d["images_u8"].shape[0])
    cams = [P.Camera(c.rotation, c.translation, c.fx * W / c.width, c.fx * W / c.width,
                     0.5 * W, 0.5 * H, W, H) for c in ds.cameras[:2]]
    rng = np.random.default_rng(11)
    gt = (rng.integers(0, 256, (2, H, W, 3)).astype(np.float64) / 255.0).astype(np.float32)
    init = _init(d)
    cfg = P.TrainConfig(iterations=2, densify=False, eval_interval=0)
    tr = Trainer(P.to_device_cloud(init), W, H, cfg, ds.scene_extent)
    tr.r.keep_grad2d = True
    ocfg = T.Config(iterations=2, eval_interval=0, seed=0)
    names = P.PARAM_NAMES
    for it in (1, 2):
        params = {k: getattr(tr.cloud, k).cpu().numpy().copy() for k in names}
        state = {k: {"m": tr.m[k].cpu().numpy().copy(), "v": tr.v[k].cpu().numpy().copy()}
                 for k in names}
        pre = {k: params[k].copy() for k in names}
        pre_state = {k: {"m": state[k]["m"].copy(), "v": state[k]["v"].copy()} for k in names}
        tr.step(it, cams[it - 1], torch.from_numpy(gt[it - 1]).cuda())
        torch.cuda.synchronize()
        n = params["positions"].shape[0]
        oloss, det = T.iteration(params, state, np.zeros(n, np.int64), np.zeros(n), 1, it,
                                 cams[it - 1], gt[it - 1], ocfg, ds.scene_extent)
        got = float(tr.loss_dev[it])
        assert abs(got - oloss) / oloss <= 2e-5, (got, oloss)
        vis = det["visible"]
        assert vis.shape[0] > 1000
        rank_of = tr.r.rank_of.cpu().numpy()
        assert int((rank_of >= 0).sum()) == vis.shape[0] and np.all(rank_of[vis] >= 0)
        g2d = tr.r.grad2d.cpu().numpy()[rank_of[vis]]
        for k, cols in (("dmean", slice(0, 2)), ("dconic", slice(2, 5)),
                        ("dcolor", slice(5, 8)), ("dopac", slice(8, 9))):
            a = g2d[:, cols].ravel()
            b = det["grad2d"][k][vis].reshape(vis.shape[0], -1).ravel()
            assert np.linalg.norm(a - b) <= 1e-3 * max(np.linalg.norm(b), 1e-300), k
        for k in names:
            a, b = tr.grads[k].cpu().numpy().ravel(), det["param_grads"][k].ravel()
            assert np.linalg.norm(a - b) <= 1e-3 * max(np.linalg.norm(b), 1e-300), k
        O.adam_step(pre, {k: tr.grads[k].cpu().numpy() for k in names}, pre_state, it, det["lrs"])
        for k in names:
            np.testing.assert_array_equal(getattr(tr.cloud, k).cpu().numpy(), pre[k], err_msg=k)


def test_backward_two_entries_per_step_is_bitwise():
    """bwd_kernel<..., 3> (three list entries per step, chosen per launch for
    launches of about one wave) == one entry per step: losses, parameters and
    Adam moments bitwise over 4 iterations."""
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200 import engine as E
    from paper_2509_05216_b200.engine import Trainer
    d = load("config1")
    ds = _dataset(d, "images_u8", d["images_u8"].shape[0])
    cfg = P.TrainConfig(iterations=4, densify=False, seed=0)
    gt = _images(ds)
    sched = P.build_schedule(4, ds.view_count, 0)
    saved = E.UNROLL2_TILES, E.CHUNK
    runs = []
    try:
        for u in (1 << 30, 0):
            E.UNROLL2_TILES, E.CHUNK = u, 0  # unchunked launches (config 1 chunks by default)
            t = Trainer(P.to_device_cloud(_init(d)), ds.width, ds.height, cfg, ds.scene_extent)
            for it in range(1, 5):
                t.step(it, ds.cameras[sched[it - 1]], gt[sched[it - 1]])
            torch.cuda.synchronize()
            assert (t.r.chunks is not None and t.r.chunks.unroll2 == 1) == bool(u)
            runs.append(t)
    finally:
        E.UNROLL2_TILES, E.CHUNK = saved
    a, b = runs
    assert torch.equal(a.loss_dev, b.loss_dev)
    for k in P.PARAM_NAMES:
        assert torch.equal(getattr(a.cloud, k), getattr(b.cloud, k)), k
        assert torch.equal(a.m[k], b.m[k]) and torch.equal(a.v[k], b.v[k]), k
