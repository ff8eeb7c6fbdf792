"""Densification (clone / split / prune) against the reference's own outputs
(tests/golden/densify.npz and train_densify.npz, made by make_golden.py
--densify from isosplat.training.densify_and_prune and train_single).

Bars: the row classification and the kept / cloned / split / pruned index
lists are exact; every output parameter is bit-identical except split
children's positions and log-scales, which pass through numpy's float64 exp
(whose SIMD dispatch can differ by 1 ulp between hosts) and are compared at
1e-6 relative.  The training run with densification active reproduces the
reference's Gaussian counts exactly and its losses within float32 tolerance.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from golden_io import cam_from, cloud_from, load


def _stats(d, device):
    from paper_2509_05216_b200.training import TrainStats
    return TrainStats(grad_accum=torch.from_numpy(d["grad_accum"]).to(device),
                      seen=torch.from_numpy(d["seen"]).to(device))


def _run(device):
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200.gaussians import GaussianCloud
    d = load("densify")
    src = cloud_from(d, "in_")
    cloud = GaussianCloud(*(torch.from_numpy(np.ascontiguousarray(getattr(src, k))).to(device)
                            for k in P.PARAM_NAMES), degree=int(src.degree))
    cfg = P.TrainConfig(seed=int(d["seed"]), opacity_prune=0.005)
    new, mp = P.densify_and_prune(cloud, _stats(d, device), cfg, int(d["iteration"]),
                                  float(d["grad_thr"]), float(d["split_thr"]),
                                  global_ids=d["gids"])
    return d, new, mp


def _check(d, new, mp):
    import paper_2509_05216_b200 as P
    for name, key in (("kept", "kept"), ("cloned", "cloned"), ("split", "split"),
                      ("pruned", "pruned")):
        assert np.array_equal(getattr(mp, name).cpu().numpy(), d[key]), name
    n_plain = d["kept"].size + d["cloned"].size
    for k in P.PARAM_NAMES:
        got = getattr(new, k).cpu().numpy()
        want = d["out_" + k]
        assert got.shape == want.shape, k
        assert np.array_equal(got[:n_plain], want[:n_plain]), k
        if k in ("positions", "log_scales"):
            np.testing.assert_allclose(got[n_plain:], want[n_plain:], rtol=1e-6, atol=1e-7)
        else:
            assert np.array_equal(got[n_plain:], want[n_plain:]), k


def test_densify_host_logic_cpu():
    """Classification, ordering and child sampling (host logic) on CPU tensors."""
    d, new, mp = _run(torch.device("cpu"))
    _check(d, new, mp)


@pytest.mark.gpu
def test_densify_matches_reference_gpu():
    d, new, mp = _run(torch.device("cuda", 0))
    _check(d, new, mp)


@pytest.mark.gpu
def test_train_with_densify_matches_reference():
    import paper_2509_05216_b200 as P
    d = load("train_densify")
    n_views = sum(1 for k in d if k.startswith("cam") and k.endswith("_R"))
    cams = []
    for i in range(n_views):
        c = cam_from(d, prefix=f"cam{i}_")
        cams.append(P.Camera(c.rotation, c.translation, c.fx, c.fy, c.cx, c.cy, c.width,
                             c.height))
    ds = P.TrainDataset(cameras=cams, images=d["images"],
                        points=P.PointCloud(d["points"], d["normals"]))
    cfg = P.TrainConfig(iterations=40, densify_start=10, densify_interval=10, densify_stop=30,
                        eval_interval=20, seed=0)
    cloud, rep = P.train_single(ds, cfg, init_cloud=cloud_from(d, "init_"))
    assert [r.iteration for r in rep.records] == list(d["rec_iter"])
    assert [r.gaussians for r in rep.records] == list(d["rec_gauss"])
    assert cloud.count == d["final_positions"].shape[0]
    ref = np.array(d["losses"])
    got = np.array(rep.iteration_losses)
    assert np.max(np.abs(got - ref) / ref) <= 2e-3, (got, ref)
    for r, p, s in zip(rep.records, d["rec_psnr"], d["rec_ssim"]):
        assert abs(r.psnr - p) <= 0.05 and abs(r.ssim - s) <= 2e-3, (r.psnr, p, r.ssim, s)


@pytest.mark.gpu
def test_device_classification_equals_numpy():
    """isg_densify_classify (float64, glibc-exact exp, on the device) == the
    reference's numpy classification (training.py:334-347) on 200K rows with
    thresholds placed inside the data's range, never-seen rows, and both
    with and without scale pruning."""
    from paper_2509_05216_b200.densify import _classify_device, classify
    from paper_2509_05216_b200.gaussians import GaussianCloud
    from paper_2509_05216_b200.training import TrainStats
    import paper_2509_05216_b200 as P
    rng = np.random.default_rng(11)
    n = 200_000
    ls = rng.normal(-4.0, 1.5, (n, 3)).astype(np.float32)
    lg = rng.normal(-2.0, 3.0, n).astype(np.float32)
    seen = rng.integers(0, 40, n).astype(np.int64)
    acc = np.abs(rng.normal(0.0, 2e-3, n)) * seen
    dev = torch.device("cuda", 0)
    z = lambda k: torch.zeros((n, k) if k > 1 else n, dtype=torch.float32, device=dev)
    cloud = GaussianCloud(z(3), torch.from_numpy(ls).to(dev), z(4), torch.from_numpy(lg).to(dev),
                          torch.zeros((n, 4, 3), dtype=torch.float32, device=dev), degree=1)
    stats = TrainStats(grad_accum=torch.from_numpy(acc).to(dev), seen=torch.from_numpy(seen).to(dev))
    gthr = float(np.median(acc / np.maximum(seen, 1)))
    sthr = float(np.median(np.exp(ls.astype(np.float64)).max(axis=1)))
    for scale_prune in (float("inf"), float(np.quantile(np.exp(ls.astype(np.float64)), 0.99))):
        cfg = P.TrainConfig(opacity_prune=0.005, scale_prune=scale_prune)
        keep, clone, split, prune, _ = classify(ls, lg, seen, acc, cfg.opacity_prune,
                                                cfg.scale_prune, gthr, sthr)
        cls = _classify_device(cloud, stats, cfg, gthr, sthr).cpu().numpy()
        ref = np.where(prune, 3, np.where(split, 2, np.where(clone, 1, 0)))
        assert (keep == (ref <= 1)).all()
        assert np.array_equal(cls, ref), (scale_prune, int((cls != ref).sum()))
        assert 0 < (ref == 2).sum() and 0 < (ref == 1).sum() and 0 < (ref == 3).sum()
