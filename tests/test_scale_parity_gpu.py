"""GPU parity at the BASELINE workload scales (configs 2, 3 and one view of
config 4), against the CPU oracle (oracle/, pinned bitwise to the reference
by tests/test_oracle_golden.py) on the same inputs.

The inputs are the benchmark's own: the gyroid isosurface points of the named
config (extract_isosurface_points, GPU, bit-exact), the reference's 3-NN scale
init, the 448-view orbit, GT = quantize8(raycast_isosurface) for the views
the schedule visits.  Reference semantics: src/rasterizer.py:105-191 (project,
lexsort, tile lists), src/_kernels.py:26-374 (projection, composite,
backward), src/metrics.py:135-189 (loss), src/engine.py:481-537 (one training
iteration), src/optim.py:20-56 (Adam).

Bars (stated per quantity; float32 production kernels vs the float64 oracle):
  * projection columns, depth order, tile offsets and entries: BIT-EXACT;
  * training lists (isg_bin_emit_live): per tile an ordered sublist of the
    reference's list, every live slot in exactly one list;
  * image: |err| <= IMG_TOL_MOST on >= 99.9 % of the values, <= IMG_TOL_MAX
    everywhere (float32 transmittance over ~1000 pairs per pixel, and
    alpha-threshold decisions that may flip at 1/255 or the 1e-4 stop);
  * loss (float32 kernel vs float64 oracle on the same image): rel <= 1e-5;
  * parameter gradients (render_backward) and the training step's 2-D
    gradients: relative L2 error <= GRAD_L2 per array, and max |err| <=
    GRAD_TOL of the array's max |value| (the composite's cancelling term
    dalpha = w T - Q / (1 - alpha) in float32 over ~1000 pairs per pixel);
  * each of 3 training iterations, both sides started from the GPU's
    pre-step state: loss rel <= 2e-5; 2-D and parameter gradients and Adam
    moments as the gradients; post-step parameters and moments BIT-EXACT
    against the reference's Adam applied to the GPU's gradients; against the
    oracle's own step |p_gpu - p_ref| <= 0.05 lr on >= 99.9 % of the values
    (Adam's step is lr * m / sqrt(v), so a gradient error e of the same sign
    moves it by O(e lr)) and <= 2 lr everywhere (Adam's bound: a near-zero
    gradient whose float32 sign differs).  Rotations: >= 90 % -- their
    gradient is exactly zero at init (isotropic scales) and at iteration 2 is
    born from the +-lr anisotropy of step 1, so Adam's sign(g) step turns
    noise-level gradients into +-lr moves;
  * free-running 3 iterations (config 2): per-iteration loss rel <= 2e-4.
"""

from __future__ import annotations

import os
import time

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

PN = ("positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs")
IMG_TOL_MOST = 1e-4
IMG_TOL_MAX = 2e-2
GRAD_TOL = 2e-2
GRAD_L2 = 1e-3
ITERS = 3

# (config, training iterations compared; 0 = init-state view only)
CASES = [("config2", ITERS), ("config3", ITERS), ("config4", 0)]
_CACHE: dict = {}


def np_(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if not b.size:
        return 0.0
    return float(np.abs(a - b).max()) / max(float(np.abs(b).max()), 1e-300)


def grad_check(what, a, b):
    """Gradient bar: rel. L2 error (||a - b|| / ||b||) <= GRAD_L2 and max
    |a - b| <= GRAD_TOL of max |b|.  Returns the stats line."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    if not b.size:
        return
    d = np.abs(a - b)
    scale = max(float(np.abs(b).max()), 1e-300)
    l2 = float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
    mx = float(d.max()) / scale
    q = float(np.quantile(d, 0.9999)) / scale
    log(f"{what}: rel L2 {l2:.2e}, max {mx:.2e}, p99.99 {q:.2e} (of max |ref|)")
    assert l2 <= GRAD_L2, f"{what}: rel L2 {l2}"
    assert mx <= GRAD_TOL, f"{what}: max rel {mx}"


def log(*a):
    print("[scale]", *a, flush=True)


def _case(name, iters):
    """Workload + oracle results for one config (built once per module)."""
    if name in _CACHE:
        return _CACHE[name]
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200 import synthetic as S
    from paper_2509_05216_b200.training import TrainDataset, PointCloud, build_schedule
    from oracle import oracle as O
    O.build()
    dev = torch.device("cuda", 0)
    nv = S.CONFIGS[name][4]
    sched = build_schedule(max(iters, 1), nv, 0)
    t0 = time.time()
    wl = S.make_workload(name, dev, view_ids=sched, log=log)
    ext = TrainDataset(wl.cameras, np.zeros((nv, 1, 1, 3)), PointCloud(wl.points, wl.normals)).scene_extent
    init = {"positions": wl.points.astype(np.float32), "log_scales": wl.log_scales.astype(np.float32)}
    n = init["positions"].shape[0]
    init["rotations"] = np.zeros((n, 4), np.float32)
    init["rotations"][:, 0] = 1.0
    init["opacity_logits"] = np.full(n, np.log(0.1 / 0.9), dtype=np.float32)
    init["sh_coeffs"] = np.zeros((n, 4, 3), np.float32)
    gt = (wl.images_u8.cpu().numpy().astype(np.float64) / 255.0).astype(np.float32)
    c = {"name": name, "wl": wl, "sched": sched, "ext": ext, "init": init, "gt": gt,
         "cam": wl.cameras[sched[0]], "iters": iters, "O": O, "P": P}
    # oracle: projection, order and lists of the first scheduled view
    from golden_io import Cloud
    cloud = Cloud(*(init[k] for k in PN), 1)
    c["cloud_np"] = cloud
    t1 = time.time()
    ob = O.project(cloud, c["cam"])
    order = O.sort_order(ob)
    sa = O._sorted_arrays(ob, order)
    own = np.arange(ob.tiles_x * ob.tiles_y, dtype=np.int32)
    off, ent = O.build_tile_lists(sa["tile_min"], sa["tile_max"], own, ob.tiles_x, ob.tiles_y)
    c.update(ob=ob, order=order, offsets=off, entries=ent)
    log(f"{name}: N={n} M={len(ob)} E={ent.shape[0]} tiles={own.shape[0]}; workload "
        f"{t1 - t0:.1f}s, oracle project+lists {time.time() - t1:.1f}s")
    _CACHE[name] = c
    return c


def _oracle_render(c):
    if "o_img" not in c:
        O = c["O"]
        t0 = time.time()
        img, aux, order = O.render_forward(c["ob"], c["cam"].width, c["cam"].height, dtype=np.float32)
        loss, dimg = O.loss_l1_dssim(img, c["gt"][0], 0.2)
        g = O.render_backward(c["cloud_np"], c["cam"], c["ob"], order, aux, dimg.astype(np.float64))
        c.update(o_img=img, o_aux=aux, o_loss=loss, o_dimg=dimg, o_grads=g)
        log(f"{c['name']}: oracle forward+loss+backward {time.time() - t0:.1f}s")
    return c


def _device_cloud(c):
    P = c["P"]
    return P.to_device_cloud(c["cloud_np"], torch.device("cuda", 0), torch.float32)


@pytest.mark.parametrize("name,iters", CASES)
def test_keys_order_and_tile_lists_bitwise(name, iters):
    c = _case(name, iters)
    P = c["P"]
    batch = P.project(_device_cloud(c), c["cam"])
    ob = c["ob"]
    np.testing.assert_array_equal(np_(batch.indices), ob.indices)
    for k in ("depth", "mean2d", "cov2d", "conic", "color", "opacity", "tile_min", "tile_max"):
        np.testing.assert_array_equal(np_(getattr(batch, k)), getattr(ob, k), err_msg=k)
    order = P.sort_order(batch)
    np.testing.assert_array_equal(np_(order), c["order"])
    tiles = batch.tiles_x * batch.tiles_y
    off, ent = P.build_tile_lists(batch.tile_min[order], batch.tile_max[order],
                                  np.arange(tiles, dtype=np.int32), batch.tiles_x, batch.tiles_y)
    np.testing.assert_array_equal(np_(off), c["offsets"])
    np.testing.assert_array_equal(np_(ent), c["entries"])


@pytest.mark.parametrize("name,iters", CASES)
def test_training_lists_are_ordered_sublists(name, iters):
    """The training step's culled lists (engine.Rasterizer, the launches the
    bench times) vs the reference's full lists of the same view."""
    c = _case(name, iters)
    P = c["P"]
    from paper_2509_05216_b200.engine import Trainer
    cfg = P.TrainConfig(iterations=1, densify=False, eval_interval=0)
    t = Trainer(_device_cloud(c), c["cam"].width, c["cam"].height, cfg, c["ext"])
    ctx = t.r.forward(t.cloud, c["cam"])
    torch.cuda.synchronize()
    off = t.r.offsets.cpu().numpy().astype(np.int64)
    slots = t.r.entries[:int(off[-1])].cpu().numpy()
    assert np.array_equal(np.sort(slots), np.arange(ctx.e)), "live slots not a permutation"
    ent = t.r.slot_rank[:ctx.e].cpu().numpy()[slots]  # live-only lists hold slots
    roff, rent = c["offsets"], c["entries"]
    assert off.shape == roff.shape
    # tile id of every entry of both lists; (tile, rank) pairs sorted by tile
    # then rank are unique, so "ordered sublist" == "subset" + per-tile ascending
    T = off.shape[0] - 1
    tid = np.repeat(np.arange(T, dtype=np.int64), np.diff(off))
    rtid = np.repeat(np.arange(T, dtype=np.int64), np.diff(roff))
    m = int(c["order"].shape[0])
    key = tid * m + ent
    rkey = rtid * m + rent
    assert np.all(np.diff(key) > 0), "training lists not rank-ascending per tile"
    assert np.all(np.diff(rkey) > 0)
    assert np.all(np.isin(key, rkey, assume_unique=True)), "training list holds a pair the reference lacks"
    log(f"{name}: training lists keep {key.size} of {rkey.size} pairs "
        f"({100.0 * (1 - key.size / rkey.size):.1f} % culled)")


@pytest.mark.parametrize("name,iters", CASES)
def test_image_loss_and_gradients(name, iters):
    c = _oracle_render(_case(name, iters))
    P = c["P"]
    cam = c["cam"]
    cloud = _device_cloud(c)
    batch = P.project(cloud, cam)
    img, aux, order = P.render_forward(batch, cam.width, cam.height, (1.0, 1.0, 1.0),
                                       dtype=torch.float32)
    err = np.abs(np_(img).astype(np.float64) - c["o_img"].astype(np.float64))
    frac = float(np.mean(err <= IMG_TOL_MOST))
    log(f"{name}: image |err| max {err.max():.2e}, p99.9 {np.quantile(err, 0.999):.2e}, "
        f"within {IMG_TOL_MOST:g}: {100 * frac:.4f} %")
    assert frac >= 0.999 and err.max() <= IMG_TOL_MAX
    # the f32 loss kernel vs the f64 oracle on the same (GPU) image
    gimg = np_(img)
    loss, dimg = P.loss_l1_dssim(gimg, c["gt"][0], 0.2)
    oloss, odimg = c["O"].loss_l1_dssim(gimg, c["gt"][0], 0.2)
    lrel = abs(loss - oloss) / abs(oloss)
    log(f"{name}: loss {loss:.9f} oracle {oloss:.9f} rel {lrel:.2e}; oracle-image loss "
        f"{c['o_loss']:.9f}; dL/dimg rel {rel_err(np_(dimg), odimg):.2e}")
    assert lrel <= 1e-5
    assert rel_err(np_(dimg), odimg) <= 2e-4
    # parameter gradients from the oracle's dL/dimage through both backwards
    g = P.render_backward(cloud, cam, batch, order, aux, c["o_dimg"].astype(np.float32))
    for k in PN:
        grad_check(f"{name}: grad {k}", np_(getattr(g, k)), getattr(c["o_grads"], k))


def _host_state(tr):
    params = {k: np_(getattr(tr.cloud, k)).copy() for k in PN}
    state = {k: {"m": np_(tr.m[k]).copy(), "v": np_(tr.v[k]).copy()} for k in PN}
    return params, state


@pytest.mark.parametrize("name,iters", [x for x in CASES if x[1] > 0])
def test_training_steps_match_oracle_from_the_same_state(name, iters):
    """Trainer.step (the benchmarked launches) vs one oracle training
    iteration (src/engine.py:481-537: render, loss, backward, ascending-tile
    fold, chain, Adam) started from the GPU's own pre-step state (parameters
    and Adam moments), for each of `iters` consecutive iterations: loss, 2-D
    gradients, parameter gradients, post-step parameters and moments.

    Starting both sides from the same state isolates one step's error; a
    free-running comparison compounds Adam's sign(g) first step, where any
    near-zero gradient whose float32 sign differs moves a parameter by 2 lr and
    changes every later gradient of that Gaussian (that trajectory's losses are
    compared in test_training_trajectory_losses)."""
    c = _case(name, iters)
    P = c["P"]
    from oracle import train as T
    from paper_2509_05216_b200.engine import Trainer
    cfg = P.TrainConfig(iterations=iters, densify=False, eval_interval=0)
    tr = Trainer(_device_cloud(c), c["cam"].width, c["cam"].height, cfg, c["ext"])
    tr.r.keep_grad2d = True  # the fused fold + chain also stores the 2-D gradients
    wl = c["wl"]
    ocfg = T.Config(iterations=iters, eval_interval=0, seed=0)
    for it in range(1, iters + 1):
        cam = wl.cameras[c["sched"][it - 1]]
        params, state = _host_state(tr)
        pre = {k: params[k].copy() for k in PN}
        pre_state = {k: {"m": state[k]["m"].copy(), "v": state[k]["v"].copy()} for k in PN}
        tr.step(it, cam, wl.images_u8[it - 1])
        torch.cuda.synchronize()
        n = params["positions"].shape[0]
        t0 = time.time()
        oloss, det = T.iteration(params, state, np.zeros(n, np.int64), np.zeros(n), 1, it, cam,
                                 c["gt"][it - 1], ocfg, c["ext"])
        got = float(tr.loss_dev[it])
        lrel = abs(got - oloss) / oloss
        log(f"{name} it {it}: oracle iteration {time.time() - t0:.1f}s; loss {got:.9f} "
            f"oracle {oloss:.9f} rel {lrel:.2e}")
        assert lrel <= 2e-5
        vis = det["visible"]
        rank_of = tr.r.rank_of.cpu().numpy()
        assert np.all(rank_of[vis] >= 0)
        assert int((rank_of >= 0).sum()) == vis.shape[0]
        g2d = tr.r.grad2d.cpu().numpy()[rank_of[vis]]
        for k, cols in (("dmean", slice(0, 2)), ("dconic", slice(2, 5)),
                        ("dcolor", slice(5, 8)), ("dopac", slice(8, 9))):
            grad_check(f"{name} it {it}: 2-D {k}", g2d[:, cols],
                       det["grad2d"][k][vis].reshape(vis.shape[0], -1))
        for k in PN:
            grad_check(f"{name} it {it}: param grad {k}", np_(tr.grads[k]), det["param_grads"][k])
        # (a) the GPU's post-step state == the reference's Adam applied to the
        # GPU's own gradients from the same pre-step state, bit for bit
        pa = {k: pre[k].copy() for k in PN}
        sa = {k: {"m": pre_state[k]["m"].copy(), "v": pre_state[k]["v"].copy()} for k in PN}
        c["O"].adam_step(pa, {k: np_(tr.grads[k]) for k in PN}, sa, it, det["lrs"])
        for k in PN:
            np.testing.assert_array_equal(np_(getattr(tr.cloud, k)), pa[k], err_msg=k)
            np.testing.assert_array_equal(np_(tr.m[k]), sa[k]["m"], err_msg=k)
            np.testing.assert_array_equal(np_(tr.v[k]), sa[k]["v"], err_msg=k)
        # (b) against the oracle's own step (its float64 gradients)
        for k in PN:
            lr = det["lrs"][k]
            a = np_(getattr(tr.cloud, k))
            d = np.abs(a.astype(np.float64) - params[k].astype(np.float64))
            close = float(np.mean(d <= 0.05 * lr))
            log(f"{name} it {it}: params {k}: max |d| {d.max() / lr:.3f} lr, "
                f"within 0.05 lr: {100 * close:.4f} %")
            assert close >= (0.9 if k == "rotations" else 0.999), k
            assert d.max() <= 2.0 * lr + 4 * float(np.spacing(np.abs(a).max())), k
            for mv in ("m", "v"):
                grad_check(f"{name} it {it}: adam {mv} {k}", np_(getattr(tr, mv)[k]),
                           state[k][mv])


def test_training_trajectory_losses():
    """Config 2, free-running: the losses of 3 GPU training iterations vs
    the oracle's own 3 iterations from the same initial state."""
    name, iters = "config2", ITERS
    c = _case(name, iters)
    P = c["P"]
    from oracle import train as T
    from paper_2509_05216_b200.engine import Trainer
    cfg = P.TrainConfig(iterations=iters, densify=False, eval_interval=0)
    tr = Trainer(_device_cloud(c), c["cam"].width, c["cam"].height, cfg, c["ext"])
    wl = c["wl"]
    for it in range(1, iters + 1):
        tr.step(it, wl.cameras[c["sched"][it - 1]], wl.images_u8[it - 1])
    ocfg = T.Config(iterations=iters, eval_interval=0, seed=0)
    cams = [wl.cameras[v] for v in c["sched"][:iters]]
    res = T.train_w1(c["gt"][:iters], cams, c["init"], ocfg, extent=c["ext"],
                     evaluate_views=False, schedule=list(range(iters)))
    got = np.array(tr.loss_dev[1:iters + 1].tolist())
    want = np.array(res.losses)
    lrel = np.abs(got - want) / want
    log(f"{name}: free-running losses {got.tolist()} oracle {want.tolist()} rel {lrel.max():.2e}")
    assert lrel.max() <= 2e-4
