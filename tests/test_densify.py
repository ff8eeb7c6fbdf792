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
