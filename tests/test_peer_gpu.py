"""The peer-store exchange under torch.distributed on the real device: one
process per GPU (torch.distributed.run), symmetric-memory receive buffers,
the pack / band-fold kernels storing into them and signal-pad barriers.
Every GPU this box offers is used (one on the round's boxes); the emulated
W=2..8 runs of the same layout are in test_dist_gpu.py / test_dist_scale_gpu.py."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_peer_exchange_multiprocess_bitwise(tmp_path):
    n = torch.cuda.device_count()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tmp_path / "peer.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(HERE, "peer_worker.py"), str(out)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-4000:]
    r = json.loads(out.read_text())
    assert r["world"] == n
    for mode in ("peer", "nccl"):
        assert r[mode]["count"] == r[mode]["ref_count"], r
        assert r[mode]["losses_equal"], r
        assert r[mode]["params_equal"], r
    assert r["peer"]["peer_capacity"] is not None
