"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the unmodified reference (isosplat 0.1.0) read-only, draws seeded
inputs with the reference's own test generators (tests/oracles.py,
tests/conftest.py) and stores inputs and outputs as small .npz fixtures next
to this script.  The fixtures travel with the repo; /root/reference does not.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from isosplat import rasterizer as R  # noqa: E402
from isosplat import metrics as Mt  # noqa: E402
from isosplat import optim as O  # noqa: E402
from isosplat import distributed as D  # noqa: E402
from isosplat.camera import OrbitSpec, make_orbit  # noqa: E402
from isosplat.gaussians import init_from_points  # noqa: E402
from isosplat.training import TrainConfig, train_single  # noqa: E402
from isosplat.engine import _build_schedule  # noqa: E402

import oracles  # noqa: E402  (reference tests/oracles.py)
from conftest import build_dataset, distance_field  # noqa: E402


def cam_dict(cam, prefix="cam_"):
    return {prefix + "R": cam.rotation, prefix + "t": cam.translation,
            prefix + "intr": np.array([cam.fx, cam.fy, cam.cx, cam.cy]),
            prefix + "size": np.array([cam.width, cam.height])}


def cloud_dict(cloud, prefix=""):
    return {prefix + "positions": cloud.positions, prefix + "log_scales": cloud.log_scales,
            prefix + "rotations": cloud.rotations,
            prefix + "opacity_logits": cloud.opacity_logits,
            prefix + "sh_coeffs": cloud.sh_coeffs, prefix + "degree": np.array(cloud.degree)}


def render_case(name, cloud, cam, bg, dl_seed, dtype=np.float64):
    batch = R.project(cloud, cam)
    order = R.sort_order(batch)
    img, aux, order2 = R.render_forward(batch, cam.width, cam.height, bg, dtype=dtype)
    assert np.array_equal(order, order2)
    rng = np.random.default_rng(dl_seed)
    dl = rng.uniform(-1.0, 1.0, img.shape).astype(img.dtype)
    cache = aux.cache
    scratch = R.backward_on_tiles(cache["sorted"], cache["own_tiles"], cache["offsets"],
                                  cache["entries"], cam.width, cam.height, cache["tiles_x"],
                                  cache["tile_size"], cache["background"], dl)
    grads = R.render_backward(cloud, cam, batch, order, aux, dl)
    out = {}
    out.update(cam_dict(cam))
    out.update(cloud_dict(cloud))
    out.update({
        "bg": np.asarray(bg, dtype=np.float64),
        "b_indices": batch.indices, "b_mean2d": batch.mean2d, "b_cov2d": batch.cov2d,
        "b_conic": batch.conic, "b_depth": batch.depth, "b_color": batch.color,
        "b_opacity": batch.opacity, "b_tile_min": batch.tile_min,
        "b_tile_max": batch.tile_max, "order": order,
        "offsets": cache["offsets"], "entries": cache["entries"],
        "image": img, "t_final": aux.t_final, "n_contrib": aux.contrib_count,
        "touch_count": aux.touch_count, "dl": dl,
        "s_dmean": scratch["dmean"], "s_dconic": scratch["dconic"],
        "s_dcolor": scratch["dcolor"], "s_dopac": scratch["dopac"],
        "grad_norm": aux.grad_norm,
        "g_positions": grads.positions, "g_log_scales": grads.log_scales,
        "g_rotations": grads.rotations, "g_opacity_logits": grads.opacity_logits,
        "g_sh_coeffs": grads.sh_coeffs,
    })
    np.savez_compressed(os.path.join(HERE, f"render_{name}.npz"), **out)
    print(f"render_{name}: N={cloud.count} M={len(batch)} E={cache['entries'].shape[0]}")


def main():
    cam = oracles.make_camera()
    render_case("random60", oracles.random_cloud(np.random.default_rng(11), 60), cam,
                oracles.BG, 1)
    render_case("fd8", oracles.fd_scene(np.random.default_rng(35), 8), cam, oracles.BG, 2)
    # Rectangular image, partial edge tiles, f32 storage and clamped colours.
    cam2 = oracles.Camera(rotation=np.eye(3), translation=np.zeros(3), fx=40.0, fy=40.0,
                          cx=27.0, cy=19.0, width=53, height=37)
    c3 = oracles.random_cloud(np.random.default_rng(12), 150)
    c3.sh_coeffs[:, 0] *= 3.0
    render_case("rect150_f32", c3, cam2, (1.0, 1.0, 1.0), 3, dtype=np.float32)

    # Isosurface scene: sphere points, reference init, an orbit view.
    grid = distance_field(24)
    ds = build_dataset(grid, 8.0, views=4, resolution=48, max_points=600)
    cloud0 = init_from_points(ds.points, degree=1)
    render_case("sphere_init", cloud0, ds.cameras[1], (1.0, 1.0, 1.0), 4, dtype=np.float32)

    # Loss on rectangular random images (f32 in -> f32 grad).
    rng = np.random.default_rng(5)
    b = rng.random((23, 31, 3)).astype(np.float32)
    a = np.clip(b + 0.1 * rng.standard_normal(b.shape), 0, 1).astype(np.float32)
    loss, grad = Mt.loss_l1_dssim(a, b, 0.2)
    img64 = rng.random((16, 19, 3))
    ref64 = rng.random((16, 19, 3))
    loss64, grad64 = Mt.loss_l1_dssim(img64, ref64, 0.35)
    np.savez_compressed(os.path.join(HERE, "loss.npz"), img=a, ref=b, loss=loss, grad=grad,
                        img64=img64, ref64=ref64, loss64=loss64, grad64=grad64,
                        ssim=Mt.ssim(a, b), psnr=Mt.psnr(a, b), w1d=Mt._W1D)

    # Adam, float32 groups, several iterations.
    rng = np.random.default_rng(6)
    params = {"positions": rng.standard_normal((7, 3)).astype(np.float32),
              "opacity_logits": rng.standard_normal(7).astype(np.float32)}
    p0 = {k: v.copy() for k, v in params.items()}
    state = O.adam_init(params)
    gs = []
    for it in range(1, 5):
        g = {k: rng.standard_normal(v.shape).astype(np.float32) for k, v in params.items()}
        gs.append(g)
        O.adam_step(params, g, state, it, {"positions": 1.6e-4 * 3.7, "opacity_logits": 5e-2})
    out = {}
    for k in params:
        out["p0_" + k] = p0[k]
        out["p_" + k] = params[k]
        out["m_" + k] = state[k]["m"]
        out["v_" + k] = state[k]["v"]
        out["g_" + k] = np.stack([g[k] for g in gs])
    np.savez_compressed(os.path.join(HERE, "adam.npz"), **out)

    # Routing mask and round-robin partition (distributed.py).
    batch = R.project(oracles.random_cloud(np.random.default_rng(13), 80), cam)
    mask = D.route_rows(batch.tile_min, batch.tile_max, 3, batch.tiles_x)
    np.savez_compressed(os.path.join(HERE, "route.npz"), tile_min=batch.tile_min,
                        tile_max=batch.tile_max, tiles_x=batch.tiles_x, mask=mask)

    # A short end-to-end training run on the reference's tiny dataset.
    tiny = build_dataset(distance_field(16), 5.0, views=4, resolution=32, max_points=48)
    cfg = TrainConfig(iterations=6, eval_interval=3, densify=False, seed=4)
    cloud, rep = train_single(tiny, cfg)
    init = init_from_points(tiny.points, degree=1)
    out = {"images": tiny.images, "points": tiny.points.positions,
           "normals": tiny.points.normals,
           "losses": np.array(rep.iteration_losses),
           "rec_iter": np.array([r.iteration for r in rep.records]),
           "rec_loss": np.array([r.loss for r in rep.records]),
           "rec_psnr": np.array([r.psnr for r in rep.records]),
           "rec_ssim": np.array([r.ssim for r in rep.records]),
           "schedule": np.array(_build_schedule(cfg.iterations, tiny.view_count, cfg.seed)),
           "scene_extent": tiny.scene_extent}
    for i, c in enumerate(tiny.cameras):
        out.update(cam_dict(c, prefix=f"cam{i}_"))
    out.update(cloud_dict(cloud, prefix="final_"))
    out.update(cloud_dict(init, prefix="init_"))
    np.savez_compressed(os.path.join(HERE, "train_tiny.npz"), **out)
    print("train_tiny losses", rep.iteration_losses)


if __name__ == "__main__" and not set(sys.argv) & {"--config1", "--densify", "--checkpoint",
                                                  "--volume"}:
    main()


def config1():
    """BASELINE config 1: sphere isosurface 20K Gaussians, 64x64, 16 views,
    100 iterations.  Stores the dataset and the reference's
    loss trajectory / final PSNR+SSIM for the PSNR-parity test."""
    import time
    grid = distance_field(128)
    ds = build_dataset(grid, 40.0, views=16, resolution=64, max_points=20000)
    cfg = TrainConfig(iterations=100, eval_interval=0, seed=0)
    t0 = time.time()
    cloud, rep = train_single(ds, cfg)
    wall = time.time() - t0
    out = {"images_u8": np.rint(ds.images * 255.0).astype(np.uint8),
           "points": ds.points.positions, "normals": ds.points.normals,
           "losses": np.array(rep.iteration_losses),
           "rec_iter": np.array([r.iteration for r in rep.records]),
           "rec_loss": np.array([r.loss for r in rep.records]),
           "rec_psnr": np.array([r.psnr for r in rep.records]),
           "rec_ssim": np.array([r.ssim for r in rep.records]),
           "total_wall_s": rep.total_wall_s, "scene_extent": ds.scene_extent,
           "init_log_scales": init_from_points(ds.points, degree=1).log_scales}
    for i, c in enumerate(ds.cameras):
        out.update(cam_dict(c, prefix=f"cam{i}_"))
    np.savez_compressed(os.path.join(HERE, "config1.npz"), **out)
    print("config1", rep.records[0].psnr, "->", rep.records[-1].psnr,
          "ssim", rep.records[-1].ssim, "wall", wall)


if __name__ == "__main__" and "--config1" in sys.argv:
    config1()


def densify():
    """densify_and_prune pinned on its own (training.py:315-389, clone + split
    + prune with child sampling seeded by (seed, iteration, global id)), and a
    short training run with densification active (engine.py:540-545)."""
    from isosplat.training import TrainStats, densify_and_prune
    grid = distance_field(24)
    ds = build_dataset(grid, 8.0, views=8, resolution=48, max_points=600)
    cloud = init_from_points(ds.points, degree=1)
    n = cloud.count
    rng = np.random.default_rng(21)
    cloud.opacity_logits[rng.random(n) < 0.1] = -7.0           # prune candidates
    cloud.log_scales += rng.normal(0.0, 0.3, cloud.log_scales.shape).astype(np.float32)
    q = rng.standard_normal((n, 4)).astype(np.float32)
    cloud.rotations[:] = q
    stats = TrainStats(grad_accum=rng.exponential(1.0, n), seen=rng.integers(0, 6, n))
    avg = stats.grad_accum / np.maximum(stats.seen, 1)
    grad_thr = float(np.quantile(avg, 0.6))
    max_scale = np.exp(cloud.log_scales.astype(np.float64)).max(axis=1)
    split_thr = float(np.median(max_scale))
    cfg = TrainConfig(seed=3, opacity_prune=0.005)
    gids = (np.arange(n, dtype=np.int64) * 3 + 1)
    new, mp = densify_and_prune(cloud, stats, cfg, 7, grad_threshold=grad_thr,
                                split_threshold=split_thr, global_ids=gids)
    out = {"seen": stats.seen, "grad_accum": stats.grad_accum, "grad_thr": grad_thr,
           "split_thr": split_thr, "gids": gids, "seed": 3, "iteration": 7,
           "kept": mp.kept, "cloned": mp.cloned, "split": mp.split, "pruned": mp.pruned}
    out.update(cloud_dict(cloud, prefix="in_"))
    out.update(cloud_dict(new, prefix="out_"))
    np.savez_compressed(os.path.join(HERE, "densify.npz"), **out)
    print("densify unit:", n, "->", new.count, "kept", mp.kept.size, "clone", mp.cloned.size,
          "split", mp.split.size, "prune", mp.pruned.size)

    cfg = TrainConfig(iterations=40, densify_start=10, densify_interval=10, densify_stop=30,
                      eval_interval=20, seed=0)
    cloud, rep = train_single(ds, cfg)
    init = init_from_points(ds.points, degree=1)
    out = {"images": ds.images, "points": ds.points.positions, "normals": ds.points.normals,
           "losses": np.array(rep.iteration_losses),
           "rec_iter": np.array([r.iteration for r in rep.records]),
           "rec_psnr": np.array([r.psnr for r in rep.records]),
           "rec_ssim": np.array([r.ssim for r in rep.records]),
           "rec_gauss": np.array([r.gaussians for r in rep.records]),
           "scene_extent": ds.scene_extent}
    for i, c in enumerate(ds.cameras):
        out.update(cam_dict(c, prefix=f"cam{i}_"))
    out.update(cloud_dict(cloud, prefix="final_"))
    out.update(cloud_dict(init, prefix="init_"))
    np.savez_compressed(os.path.join(HERE, "train_densify.npz"), **out)
    print("train_densify:", init.count, "->", cloud.count, "records",
          [(r.iteration, r.gaussians, round(r.psnr, 3)) for r in rep.records])


if __name__ == "__main__" and "--densify" in sys.argv:
    densify()


def checkpoint():
    """SSGC checkpoint bytes (gaussians.py:194-204) of a seeded random cloud."""
    from isosplat.gaussians import save_checkpoint
    c = oracles.random_cloud(np.random.default_rng(31), 40)
    save_checkpoint(os.path.join(HERE, "ckpt_random40.ssgc"), c)
    np.savez_compressed(os.path.join(HERE, "ckpt_random40.npz"), **cloud_dict(c))


if __name__ == "__main__" and "--checkpoint" in sys.argv:
    checkpoint()


def volume():
    """Dataset generation (volume.py, raycast.py): point extraction (plain,
    strided + subsampled) and raycast views of a small gyroid and sphere."""
    from isosplat.raycast import raycast_isosurface
    from isosplat.volume import VolumeGrid, extract_isosurface_points
    out = {}
    n, periods = 28, 2.0
    s = 2.0 * np.pi * periods / (n - 1)
    ax = np.arange(n, dtype=np.float64) * s
    sx, cx = np.sin(ax), np.cos(ax)
    data = (sx[None, None, :] * cx[None, :, None] + sx[None, :, None] * cx[:, None, None]
            + sx[:, None, None] * cx[None, None, :])
    gyr = VolumeGrid(dims=(n, n, n), spacing=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0), data=data)
    # anisotropic spacing / offset origin on the sphere
    sph0 = distance_field(20)
    sph = VolumeGrid(dims=sph0.dims, spacing=(0.5, 0.75, 1.0), origin=(-1.0, 2.0, 0.5),
                     data=sph0.data)
    for tag, grid, iso in (("gyr", gyr, 0.0), ("sph", sph, 6.0)):
        out[tag + "_data"] = grid.data
        out[tag + "_spacing"] = np.asarray(grid.spacing)
        out[tag + "_origin"] = np.asarray(grid.origin)
        out[tag + "_iso"] = np.array(iso)
        pc = extract_isosurface_points(grid, iso)
        out[tag + "_pos"], out[tag + "_nrm"] = pc.positions, pc.normals
        pc2 = extract_isosurface_points(grid, iso, stride=2, max_points=150, seed=3)
        out[tag + "_pos_s2"], out[tag + "_nrm_s2"] = pc2.positions, pc2.normals
        lo = np.asarray(grid.world_min)
        hi = np.asarray(grid.world_max)
        spec = OrbitSpec(count=3, center=tuple((lo + hi) / 2.0),
                         radius=1.5 * float(np.linalg.norm(hi - lo) / 2.0), width=40, height=34)
        for i, cam in enumerate(make_orbit(spec)):
            out.update(cam_dict(cam, f"{tag}_cam{i}_"))
            out[f"{tag}_img{i}"] = raycast_isosurface(grid, iso, cam)
    # a camera inside the volume and a coarse step with few refinements
    cam = make_orbit(OrbitSpec(count=2, center=(13.5, 13.5, 13.5), radius=6.0, width=24,
                               height=24))[1]
    out.update(cam_dict(cam, "gyr_in_"))
    out["gyr_in_img"] = raycast_isosurface(gyr, 0.0, cam, step_scale=1.5, refine_steps=3)
    np.savez_compressed(os.path.join(HERE, "volume.npz"), **out)


if __name__ == "__main__" and "--volume" in sys.argv:
    volume()
