"""Pin the CPU oracle (oracle/isg_oracle.c) to the reference's own outputs.

The fixtures in tests/golden/ were produced by running the unmodified
reference (tests/golden/make_golden.py).  The oracle restates the reference
in left-to-right float64 C without FMA, so every integer/index output must
match bit for bit and so must the float outputs of the projection, the
composite, the backward scratch, the chain rule and Adam.
"""

from __future__ import annotations

import numpy as np
import pytest

from golden_io import RENDER_CASES, cam_from, cloud_from, load


@pytest.mark.parametrize("case", RENDER_CASES)
def test_project_bitwise(orc, case):
    d = load("render_" + case)
    batch = orc.project(cloud_from(d), cam_from(d))
    np.testing.assert_array_equal(batch.indices, d["b_indices"])
    for k in ("mean2d", "cov2d", "conic", "depth", "color", "opacity", "tile_min", "tile_max"):
        np.testing.assert_array_equal(getattr(batch, k), d["b_" + k], err_msg=k)


@pytest.mark.parametrize("case", RENDER_CASES)
def test_sort_and_tile_lists_bitwise(orc, case):
    d = load("render_" + case)
    batch = orc.project(cloud_from(d), cam_from(d))
    order = orc.sort_order(batch)
    np.testing.assert_array_equal(order, d["order"])
    offsets, entries = orc.build_tile_lists(
        batch.tile_min[order], batch.tile_max[order],
        np.arange(batch.tiles_x * batch.tiles_y, dtype=np.int32), batch.tiles_x, batch.tiles_y)
    np.testing.assert_array_equal(offsets, d["offsets"])
    np.testing.assert_array_equal(entries, d["entries"])


@pytest.mark.parametrize("case", RENDER_CASES)
def test_forward_backward_chain_bitwise(orc, case):
    d = load("render_" + case)
    cloud, cam = cloud_from(d), cam_from(d)
    batch = orc.project(cloud, cam)
    img, aux, order = orc.render_forward(batch, cam.width, cam.height, tuple(d["bg"]),
                                         dtype=d["image"].dtype)
    np.testing.assert_array_equal(img, d["image"])
    np.testing.assert_array_equal(aux.t_final, d["t_final"])
    np.testing.assert_array_equal(aux.contrib_count, d["n_contrib"])
    np.testing.assert_array_equal(aux.touch_count, d["touch_count"])
    c = aux.cache
    scratch = orc.backward_on_tiles(c["sorted"], c["own_tiles"], c["offsets"], c["entries"],
                                    cam.width, cam.height, c["tiles_x"], c["tile_size"],
                                    c["background"], d["dl"])
    for k in ("dmean", "dconic", "dcolor", "dopac"):
        np.testing.assert_array_equal(scratch[k], d["s_" + k], err_msg=k)
    grads = orc.render_backward(cloud, cam, batch, order, aux, d["dl"])
    np.testing.assert_array_equal(aux.grad_norm, d["grad_norm"])
    for k in ("positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs"):
        np.testing.assert_array_equal(getattr(grads, k), d["g_" + k], err_msg=k)


def test_loss_bitwise(orc):
    d = load("loss")
    loss, grad = orc.loss_l1_dssim(d["img"], d["ref"], 0.2)
    assert loss == float(d["loss"])
    assert grad.dtype == np.float32
    np.testing.assert_array_equal(grad, d["grad"])
    loss64, grad64 = orc.loss_l1_dssim(d["img64"], d["ref64"], 0.35)
    assert loss64 == float(d["loss64"])
    np.testing.assert_array_equal(grad64, d["grad64"])
    assert orc.ssim(d["img"], d["ref"]) == float(d["ssim"])
    assert orc.psnr(d["img"], d["ref"]) == float(d["psnr"])


def test_ssim_window_pinned(orc):
    # The 11-tap window hard-coded in the oracle (and the CUDA loss) is the
    # reference's metrics._W1D, bit for bit.
    d = load("loss")
    import re
    src = open(__import__("os").path.join(orc._HERE, "isg_oracle.c")).read()
    block = src[src.index("W1D[11]"):]
    hexes = re.findall(r"0x1\.[0-9a-f]+p-\d+", block)[:11]
    np.testing.assert_array_equal(np.array([float.fromhex(h) for h in hexes]), d["w1d"])


def test_adam_bitwise(orc):
    d = load("adam")
    names = ["positions", "opacity_logits"]
    params = {k: d["p0_" + k].copy() for k in names}
    state = {k: {"m": np.zeros_like(params[k]), "v": np.zeros_like(params[k])} for k in names}
    for it in range(1, 5):
        g = {k: d["g_" + k][it - 1] for k in names}
        orc.adam_step(params, g, state, it, {"positions": 1.6e-4 * 3.7, "opacity_logits": 5e-2})
    for k in names:
        np.testing.assert_array_equal(params[k], d["p_" + k])
        np.testing.assert_array_equal(state[k]["m"], d["m_" + k])
        np.testing.assert_array_equal(state[k]["v"], d["v_" + k])


def test_route_mask(orc):
    d = load("route")
    mask = orc.route_mask(d["tile_min"], d["tile_max"], 3, int(d["tiles_x"]))
    np.testing.assert_array_equal(mask, d["mask"])


def _cams(d, count):
    from golden_io import cam_from
    return [cam_from(d, prefix=f"cam{i}_") for i in range(count)]


def test_train_loop_tiny_bitwise(orc):
    """The oracle's W=1 loop reproduces the reference run (6 its, eval at 3, 6)."""
    from oracle import train as T
    d = load("train_tiny")
    cams = _cams(d, d["images"].shape[0])
    assert T.build_schedule(6, len(cams), 4) == list(d["schedule"])
    assert T.scene_extent(cams) == float(d["scene_extent"])
    init = {k: d["init_" + k] for k in T.PARAM_NAMES}
    cfg = T.Config(iterations=6, eval_interval=3, seed=4)
    res = T.train_w1(d["images"], cams, init, cfg)
    assert res.losses == list(d["losses"])
    assert [r.iteration for r in res.records] == list(d["rec_iter"])
    assert [r.loss for r in res.records] == list(d["rec_loss"])
    assert [r.psnr for r in res.records] == list(d["rec_psnr"])
    assert [r.ssim for r in res.records] == list(d["rec_ssim"])
    for k in T.PARAM_NAMES:
        np.testing.assert_array_equal(res.params[k], d["final_" + k], err_msg=k)


def test_train_loop_config1_bitwise(orc):
    """BASELINE config 1 (sphere 20K G, 64^2, 16 views, 100 its): the oracle
    reproduces the reference's loss trajectory and final PSNR/SSIM bitwise."""
    from oracle import train as T
    d = load("config1")
    cams = _cams(d, d["images_u8"].shape[0])
    images = (d["images_u8"].astype(np.float64) / 255.0).astype(np.float32)
    pts = d["points"]
    init = init_params_from(pts, d["init_log_scales"])
    cfg = T.Config(iterations=100, eval_interval=0, seed=0)
    res = T.train_w1(images, cams, init, cfg)
    assert res.losses == list(d["losses"])
    assert [r.psnr for r in res.records] == list(d["rec_psnr"])
    assert [r.ssim for r in res.records] == list(d["rec_ssim"])


def init_params_from(points, log_scales, degree=1):
    """gaussians.py:165-191 with the kNN scales taken from the fixture."""
    n = points.shape[0]
    k = (degree + 1) ** 2
    rot = np.zeros((n, 4), dtype=np.float32)
    rot[:, 0] = 1.0
    import math
    return {"positions": points.astype(np.float32), "log_scales": np.asarray(log_scales, np.float32),
            "rotations": rot,
            "opacity_logits": np.full(n, math.log(0.1 / 0.9), dtype=np.float32),
            "sh_coeffs": np.zeros((n, k, 3), dtype=np.float32)}
