"""GPU parity: the CUDA path (libisogs.so through the package API) against the
reference's own outputs (tests/golden/, produced by running the reference)
and the CPU oracle (oracle/).

Bars, stated per quantity:
  * projection (depth, mean2d, cov2d, conic, colour, opacity, tile rect), sort
    order, per-tile offsets and entries: BIT-EXACT;
  * float64 build: composite image, T_final, n_contrib, touch counts:
    BIT-EXACT; backward scratch and parameter gradients: rel. err <= 1e-9 of
    each array's max |value| (the GPU sums the 256 pixels of a tile as a tree,
    the reference sequentially);
  * float32 build (production): image |err| <= 2e-5 on >= 99.9% of pixels and
    <= 5e-3 everywhere (alpha-threshold decisions may flip near 1/255 or the
    1e-4 stop); parameter gradients rel. err <= 2e-3 of max |value| per array;
  * loss: float64 rel. err <= 1e-12, float32 <= 1e-5; Adam: BIT-EXACT.
"""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

from golden_io import RENDER_CASES, cam_from, cloud_from, load

pytestmark = pytest.mark.gpu

PN = ("positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs")


@pytest.fixture(scope="module")
def P():
    import paper_2509_05216_b200 as pkg
    from paper_2509_05216_b200 import _lib
    _lib.require_cuda()
    return pkg


def np_(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(float(np.abs(b).max()) if b.size else 0.0, 1e-300)
    return float(np.abs(a - b).max()) / scale if b.size else 0.0


@pytest.mark.parametrize("case", RENDER_CASES)
def test_project_bitwise(P, case):
    d = load("render_" + case)
    batch = P.project(cloud_from(d), cam_from(d))
    np.testing.assert_array_equal(np_(batch.indices), d["b_indices"])
    for k in ("mean2d", "cov2d", "conic", "depth", "color", "opacity", "tile_min", "tile_max"):
        np.testing.assert_array_equal(np_(getattr(batch, k)), d["b_" + k], err_msg=k)


@pytest.mark.parametrize("case", RENDER_CASES)
def test_sort_order_and_tile_lists_bitwise(P, case):
    d = load("render_" + case)
    batch = P.project(cloud_from(d), cam_from(d))
    order = P.sort_order(batch)
    np.testing.assert_array_equal(np_(order), d["order"])
    tiles = batch.tiles_x * batch.tiles_y
    offsets, entries = P.build_tile_lists(batch.tile_min[order], batch.tile_max[order],
                                          np.arange(tiles, dtype=np.int32), batch.tiles_x,
                                          batch.tiles_y)
    np.testing.assert_array_equal(np_(offsets), d["offsets"])
    np.testing.assert_array_equal(np_(entries), d["entries"])


def test_tile_lists_for_round_robin_subset(P, orc):
    d = load("render_random60")
    batch = orc.project(cloud_from(d), cam_from(d))
    order = orc.sort_order(batch)
    own = np.arange(1, batch.tiles_x * batch.tiles_y, 3, dtype=np.int32)
    ref_off, ref_ent = orc.build_tile_lists(batch.tile_min[order], batch.tile_max[order], own,
                                            batch.tiles_x, batch.tiles_y)
    off, ent = P.build_tile_lists(batch.tile_min[order], batch.tile_max[order], own,
                                  batch.tiles_x, batch.tiles_y)
    np.testing.assert_array_equal(np_(off), ref_off)
    np.testing.assert_array_equal(np_(ent), ref_ent)


@pytest.mark.parametrize("case", RENDER_CASES)
def test_render_forward_float64_bitwise(P, case):
    d = load("render_" + case)
    cam = cam_from(d)
    batch = P.project(cloud_from(d), cam)
    img, aux, order = P.render_forward(batch, cam.width, cam.height, tuple(d["bg"]),
                                       dtype=torch.float64)
    np.testing.assert_array_equal(np_(order), d["order"])
    np.testing.assert_array_equal(np_(img).astype(d["image"].dtype), d["image"])
    np.testing.assert_array_equal(np_(aux.t_final), d["t_final"])
    np.testing.assert_array_equal(np_(aux.contrib_count), d["n_contrib"])
    np.testing.assert_array_equal(np_(aux.touch_count), d["touch_count"])


@pytest.mark.parametrize("case", RENDER_CASES)
def test_render_forward_float32_tolerance(P, case):
    d = load("render_" + case)
    cam = cam_from(d)
    batch = P.project(cloud_from(d), cam)
    img, aux, _ = P.render_forward(batch, cam.width, cam.height, tuple(d["bg"]),
                                   dtype=torch.float32)
    err = np.abs(np_(img).astype(np.float64) - d["image"].astype(np.float64))
    assert np.mean(err <= 2e-5) >= 0.999, float(err.max())
    assert err.max() <= 5e-3


@pytest.mark.parametrize("case", RENDER_CASES)
def test_backward_float64_tight(P, case):
    d = load("render_" + case)
    cam, cloud = cam_from(d), cloud_from(d)
    batch = P.project(cloud, cam)
    img, aux, order = P.render_forward(batch, cam.width, cam.height, tuple(d["bg"]),
                                       dtype=torch.float64)
    grads = P.render_backward(cloud, cam, batch, order, aux, d["dl"].astype(np.float64))
    for k in PN:
        assert rel_err(np_(getattr(grads, k)), d["g_" + k]) <= 1e-9, k
    assert rel_err(np_(aux.grad_norm), d["grad_norm"]) <= 1e-9


@pytest.mark.parametrize("case", RENDER_CASES)
def test_backward_on_tiles_scratch_float64(P, case):
    d = load("render_" + case)
    cam = cam_from(d)
    batch = P.project(cloud_from(d), cam)
    order = P.sort_order(batch)
    sa = {k: getattr(batch, k)[order] for k in ("mean2d", "conic", "color", "opacity")}
    own = np.arange(batch.tiles_x * batch.tiles_y, dtype=np.int32)
    scratch = P.backward_on_tiles(sa, own, d["offsets"], d["entries"], cam.width, cam.height,
                                  batch.tiles_x, 16, d["bg"], d["dl"].astype(np.float64))
    for k in ("dmean", "dconic", "dcolor", "dopac"):
        assert rel_err(np_(scratch[k]), d["s_" + k]) <= 1e-9, k


@pytest.mark.parametrize("case", RENDER_CASES)
def test_backward_float32_tolerance(P, case):
    d = load("render_" + case)
    cam, cloud = cam_from(d), cloud_from(d)
    batch = P.project(cloud, cam)
    img, aux, order = P.render_forward(batch, cam.width, cam.height, tuple(d["bg"]),
                                       dtype=torch.float32)
    grads = P.render_backward(cloud, cam, batch, order, aux, d["dl"].astype(np.float32))
    for k in PN:
        assert rel_err(np_(getattr(grads, k)), d["g_" + k]) <= 2e-3, k


@pytest.mark.parametrize("case", RENDER_CASES)
def test_chain_bitwise_given_reference_2d_grads(P, orc, case):
    d = load("render_" + case)
    cam, cloud = cam_from(d), cloud_from(d)
    m = d["b_indices"].shape[0]
    scratch = {k: d["s_" + k] for k in ("dmean", "dconic", "dcolor", "dopac")}
    acc = orc.reduce_scratch(d["entries"], scratch, m)  # sorted rows, tile order
    gpu_acc = P.reduce_scratch(d["entries"], scratch, m)
    for k in acc:
        np.testing.assert_array_equal(np_(gpu_acc[k]), acc[k], err_msg=k)
    n = cloud.count
    order = d["order"]
    flags = np.zeros(n, dtype=np.uint8)
    full = {}
    for k in acc:
        b = np.zeros_like(acc[k])
        b[order] = acc[k]
        f = np.zeros((n,) + b.shape[1:])
        f[d["b_indices"]] = b
        full[k] = f
    flags[d["b_indices"]] = 1
    grads = P.chain_to_params(cloud, cam, flags, full["dmean"], full["dconic"], full["dcolor"],
                              full["dopac"])
    for k in PN:
        np.testing.assert_array_equal(np_(getattr(grads, k)), d["g_" + k], err_msg=k)


def test_loss_parity(P):
    d = load("loss")
    loss, grad = P.loss_l1_dssim(d["img64"], d["ref64"], 0.35)
    assert abs(loss - float(d["loss64"])) <= 1e-12 * abs(float(d["loss64"]))
    assert rel_err(np_(grad), d["grad64"]) <= 1e-12
    loss32, grad32 = P.loss_l1_dssim(d["img"], d["ref"], 0.2)
    assert grad32.dtype == torch.float32
    assert abs(loss32 - float(d["loss"])) <= 1e-5 * abs(float(d["loss"]))
    assert rel_err(np_(grad32), d["grad"]) <= 2e-4
    assert abs(P.ssim(d["img"], d["ref"]) - float(d["ssim"])) <= 1e-12
    assert abs(P.psnr(d["img"], d["ref"]) - float(d["psnr"])) <= 1e-9


def test_adam_bitwise(P):
    d = load("adam")
    names = ["positions", "opacity_logits"]
    params = {k: torch.from_numpy(d["p0_" + k].copy()).cuda() for k in names}
    state = P.adam_init(params)
    for it in range(1, 5):
        g = {k: torch.from_numpy(d["g_" + k][it - 1]).cuda() for k in names}
        P.adam_step(params, g, state, it, {"positions": 1.6e-4 * 3.7, "opacity_logits": 5e-2})
    for k in names:
        np.testing.assert_array_equal(np_(params[k]), d["p_" + k])
        np.testing.assert_array_equal(np_(state[k]["m"]), d["m_" + k])
        np.testing.assert_array_equal(np_(state[k]["v"]), d["v_" + k])


def test_device_exp_is_glibc_exact(P):
    import ctypes
    from paper_2509_05216_b200 import _lib as L
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.uniform(-40, 10, 100_000), rng.uniform(-6, 0, 100_000),
                        rng.uniform(-745, -700, 20_000), rng.uniform(-800, 709, 20_000)])
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    L.check(L.lib().isg_exp_f64(x.size, L.ptr(xd), L.ptr(yd), L.stream_ptr()), "exp")
    want = np.array([math.exp(v) for v in x])
    np.testing.assert_array_equal(np_(yd), want)


def test_empty_and_offscreen(P):
    from golden_io import Cam, Cloud
    cam = Cam(np.eye(3), np.zeros(3), 45.0, 45.0, 24.0, 24.0, 48, 48)
    cloud = Cloud(np.array([[0.0, 0.0, -4.0]]), np.full((1, 3), np.log(0.1)),
                  np.array([[1.0, 0, 0, 0]]), np.array([0.0]), np.zeros((1, 4, 3)), 1)
    batch = P.project(cloud, cam)
    assert len(batch) == 0
    img, aux, order = P.render_forward(batch, 48, 48, (0.25, 0.5, 0.75), dtype=torch.float64)
    np.testing.assert_array_equal(np_(img), np.broadcast_to(np.array([0.25, 0.5, 0.75]), (48, 48, 3)))
    assert order.numel() == 0
    grads = P.render_backward(cloud, cam, batch, order, aux, np.ones((48, 48, 3)))
    assert float(np.abs(np_(grads.positions)).max()) == 0.0


def test_backward_rejects_mismatched_context(P):
    d = load("render_random60")
    cam, cloud = cam_from(d), cloud_from(d)
    batch = P.project(cloud, cam)
    img, aux, order = P.render_forward(batch, cam.width, cam.height, (1, 1, 1))
    with pytest.raises(ValueError):
        P.render_backward(cloud, cam, batch, order[:-1], aux, np.ones((48, 48, 3)))
    with pytest.raises(ValueError):
        P.render_backward(cloud, cam, batch, order, aux, np.ones((47, 48, 3)))
    with pytest.raises(ValueError):
        P.render_forward(batch, 47, 48)


def test_sort_depth_equals_full_64bit_sort():
    """isg_sort_depth (6 passes over the top 48 bits + run fix-up) is the
    stable 64-bit sort: adversarial keys with long equal-top-48 runs, exact
    duplicates and the culled ~0 tail."""
    from paper_2509_05216_b200 import _lib as L
    g = torch.Generator().manual_seed(3)
    n = 200_000
    base = torch.randint(0, 2**40, (n,), generator=g, dtype=torch.int64) << 20
    base[: n // 2] = base[: n // 2] % (2**26 << 20)  # many shared top-48 prefixes
    low = torch.randint(0, 2**16, (n,), generator=g, dtype=torch.int64)
    low[::7] = 5  # duplicates
    keys = (base | low)
    keys[-1000:] = -1  # culled (~0)
    keys[1000:3000] = keys[1000]  # a long run of identical keys
    keys = keys.cuda()
    vals = torch.arange(n, dtype=torch.int32, device="cuda")
    ws1, ws2 = L.Workspace(), L.Workspace()
    k1, v1 = L.sort_pairs(keys, vals, (0, 64), ws1)
    k2, v2 = L.sort_depth(keys, vals, ws2)
    assert torch.equal(k1, k2) and torch.equal(v1, v2)


@pytest.mark.parametrize("width,bits", [(2, (0, 15)), (2, (0, 16)), (4, (0, 14)), (4, (3, 29)),
                                        (8, (0, 64)), (8, (24, 64))])
def test_radix_sort_is_a_stable_sort(width, bits):
    """The hand-written LSD radix sort (radix.cu) == torch's stable sort on
    the same key bits: keys, and values (original positions) for ties; sizes
    with a partial last CTA and many equal digits."""
    from paper_2509_05216_b200 import _lib as L
    g = torch.Generator().manual_seed(width * 100 + bits[1])
    for n in (1, 4095, 4096, 100_003, 3_000_001):
        dt = {2: torch.int16, 4: torch.int32, 8: torch.int64}[width]
        raw = torch.randint(-2**62, 2**62, (n,), generator=g, dtype=torch.int64)
        raw[: n // 3] = raw[: n // 3] % 7  # heavy duplicates
        keys = raw.to(dt) if width < 8 else raw
        keys = keys.cuda()
        vals = torch.arange(n, dtype=torch.int32, device="cuda")
        ko, vo = L.sort_pairs(keys, vals, bits, L.Workspace())
        # reference: stable sort on the selected bits (unsigned)
        u = keys.to(torch.int64) & ((1 << (8 * width)) - 1) if width < 8 else keys
        b0, b1 = bits
        if width == 8:
            sel = (u >> b0) & ((1 << (b1 - b0)) - 1) if b1 - b0 < 64 else u
            # unsigned order of 64-bit keys: flip the sign bit
            sel = sel ^ (-2**63) if b1 - b0 == 64 else sel
        else:
            sel = (u >> b0) & ((1 << (b1 - b0)) - 1)
        _, idx = torch.sort(sel, stable=True)
        assert torch.equal(vo, idx.to(torch.int32)), (n, width, bits)
        assert torch.equal(ko, keys[idx]), (n, width, bits)


def test_depth_sort_long_reversed_run_is_bounded():
    """A 200K-key run with equal top 40 bits in reverse order of the low
    bits (the tie fix-up's worst case: heap sort, not quadratic insertion)."""
    from paper_2509_05216_b200 import _lib as L
    n = 200_000
    keys = (torch.full((n,), 0x40A00000, dtype=torch.int64) << 24) | \
        torch.arange(n - 1, -1, -1, dtype=torch.int64)
    keys = keys.cuda()
    vals = torch.arange(n, dtype=torch.int32, device="cuda")
    k2, v2 = L.sort_depth(keys, vals, L.Workspace())
    torch.cuda.synchronize()
    assert torch.equal(v2, torch.arange(n - 1, -1, -1, dtype=torch.int32, device="cuda"))
    assert bool((k2[1:] >= k2[:-1]).all())


def test_route_rows_round_robin_matches_reference():
    """route_rows(tile_min, tile_max, workers, tiles_x) on the device
    (isg_route_mask) == the reference's _route_mask output (route.npz)."""
    from paper_2509_05216_b200 import distributed as D
    d = load("route")
    mask = D.route_rows(d["tile_min"], d["tile_max"], 3, int(d["tiles_x"]))
    np.testing.assert_array_equal(np_(mask), d["mask"])


def test_gpu_knn_init_matches_reference_bitwise():
    """init_log_scales on the GPU (isg_knn_mean_grid) reproduces the
    reference's init_from_points log-scales bit for bit (config 1: 20000
    points, the reference's grid path)."""
    from paper_2509_05216_b200.training import init_log_scales
    d = load("config1")
    got = init_log_scales(d["points"])
    assert got.dtype == np.float32 and got.shape == d["init_log_scales"].shape
    assert np.array_equal(got, d["init_log_scales"])
