"""SSGC checkpoint IO against the reference's own file (tests/golden/
ckpt_random40.ssgc, written by isosplat.gaussians.save_checkpoint): byte-
identical writer, loader round trip, and the reference's validation errors.
Host-side logic (CPU tensors); the device path is the same code."""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch

from golden_io import GOLDEN, cloud_from, load


def _cpu_cloud(d):
    from paper_2509_05216_b200.gaussians import PARAM_NAMES, GaussianCloud
    c = cloud_from(d)
    return GaussianCloud(*(torch.from_numpy(np.ascontiguousarray(getattr(c, k)))
                           for k in PARAM_NAMES), degree=int(c.degree))


def test_writer_bytes_match_reference(tmp_path):
    from paper_2509_05216_b200.gaussians import save_checkpoint
    d = load("ckpt_random40")
    out = tmp_path / "a.ssgc"
    save_checkpoint(str(out), _cpu_cloud(d))
    with open(os.path.join(GOLDEN, "ckpt_random40.ssgc"), "rb") as fh:
        ref = fh.read()
    assert out.read_bytes() == ref


def test_loader_roundtrip_and_errors(tmp_path):
    from paper_2509_05216_b200.gaussians import PARAM_NAMES, load_checkpoint
    d = load("ckpt_random40")
    got = load_checkpoint(os.path.join(GOLDEN, "ckpt_random40.ssgc"), torch.device("cpu"))
    for k in PARAM_NAMES:
        assert np.array_equal(getattr(got, k).numpy(), d[k].astype(np.float32)), k
    assert got.degree == int(d["degree"])
    bad = tmp_path / "bad.ssgc"
    bad.write_bytes(b"XXXX" + bytes(20))
    with pytest.raises(ValueError, match="bad magic"):
        load_checkpoint(str(bad), torch.device("cpu"))
    with open(os.path.join(GOLDEN, "ckpt_random40.ssgc"), "rb") as fh:
        blob = fh.read()
    short = tmp_path / "short.ssgc"
    short.write_bytes(blob[:-4])
    with pytest.raises(ValueError, match="expected"):
        load_checkpoint(str(short), torch.device("cpu"))
