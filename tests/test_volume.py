"""Dataset generation (volume.py, raycast.py) against the
reference's own outputs (tests/golden/volume.npz, make_golden.py --volume).

Bars: BIT-EXACT.  Point positions and normals of extract_isosurface_points
(plain, and strided + seeded subsample) and every raycast view, including a
camera inside the volume with a coarse step and 3 refinements, equal the
reference's float64 arrays bit for bit."""

from __future__ import annotations

import numpy as np
import pytest

from golden_io import cam_from, load


def _grid(d, tag):
    from paper_2509_05216_b200.volume import VolumeGrid
    data = d[tag + "_data"]
    nz, ny, nx = data.shape
    return VolumeGrid(dims=(nx, ny, nz), spacing=tuple(d[tag + "_spacing"].tolist()),
                      origin=tuple(d[tag + "_origin"].tolist()), data=data)


def test_volume_grid_host_checks():
    from paper_2509_05216_b200.volume import VolumeGrid, distance_field, quantize8
    g = distance_field(8)
    assert g.dims == (8, 8, 8)
    np.testing.assert_array_equal(g.world_max, [7.0, 7.0, 7.0])
    with pytest.raises(ValueError):
        VolumeGrid(dims=(4, 4, 3), spacing=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0),
                   data=np.zeros((4, 4, 4)))
    with pytest.raises(ValueError):
        VolumeGrid(dims=(4, 4, 4), spacing=(1.0, 0.0, 1.0), origin=(0.0, 0.0, 0.0),
                   data=np.zeros((4, 4, 4)))
    q = quantize8(np.array([-0.1, 0.5 / 255.0, 1.5 / 255.0, 2.0]))
    np.testing.assert_array_equal(q * 255.0, [0.0, 0.0, 2.0, 255.0])  # ties to even


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["gyr", "sph"])
def test_extract_points_bitwise(tag):
    from paper_2509_05216_b200.volume import extract_isosurface_points
    d = load("volume")
    g = _grid(d, tag)
    iso = float(d[tag + "_iso"])
    pc = extract_isosurface_points(g, iso)
    assert pc.positions.shape == d[tag + "_pos"].shape
    np.testing.assert_array_equal(pc.positions, d[tag + "_pos"])
    np.testing.assert_array_equal(pc.normals, d[tag + "_nrm"])
    pc2 = extract_isosurface_points(g, iso, stride=2, max_points=150, seed=3)
    np.testing.assert_array_equal(pc2.positions, d[tag + "_pos_s2"])
    np.testing.assert_array_equal(pc2.normals, d[tag + "_nrm_s2"])
    # isovalue outside the open data range: no crossing
    assert extract_isosurface_points(g, 1e9).count == 0


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["gyr", "sph"])
def test_raycast_bitwise(tag):
    from paper_2509_05216_b200.volume import quantize8, raycast_isosurface
    d = load("volume")
    g = _grid(d, tag)
    iso = float(d[tag + "_iso"])
    for i in range(3):
        cam = cam_from(d, prefix=f"{tag}_cam{i}_")
        img = raycast_isosurface(g, iso, cam).cpu().numpy()
        want = d[f"{tag}_img{i}"]
        assert (want != 1.0).any()  # the surface is in view
        np.testing.assert_array_equal(img, want)
        codes = raycast_isosurface(g, iso, cam, codes=True).cpu().numpy()
        np.testing.assert_array_equal(codes / 255.0, quantize8(want))


@pytest.mark.gpu
def test_raycast_inside_coarse_step():
    from paper_2509_05216_b200.volume import raycast_isosurface
    d = load("volume")
    cam = cam_from(d, prefix="gyr_in_")
    img = raycast_isosurface(_grid(d, "gyr"), 0.0, cam, step_scale=1.5, refine_steps=3)
    np.testing.assert_array_equal(img.cpu().numpy(), d["gyr_in_img"])


@pytest.mark.gpu
def test_host_gyroid_points_match_device_extraction():
    """bench.py's CPU arm extracts the gyroid points with the host restatement
    (synthetic.gyroid_points); they must be the GPU arm's points exactly."""
    from paper_2509_05216_b200 import synthetic as S
    from paper_2509_05216_b200.volume import extract_isosurface_points, gyroid_grid
    pos, _ = S.gyroid_points(40, 3.0, 2000, seed=0)
    pc = extract_isosurface_points(gyroid_grid(40, 3.0), 0.0, max_points=2000, seed=0)
    np.testing.assert_array_equal(pos, pc.positions)
