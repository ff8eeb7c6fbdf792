"""bench.py's output contract (one JSON line on stdout, the keys the driver
reads), on a short config-2 run of our arm."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_has_the_contract_keys():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "config2",
                        "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--warm-iters", "0"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, p.stdout  # stdout carries only the JSON line
    d = json.loads(lines[0])
    for k, t in (("metric", str), ("value", float), ("unit", str), ("n_gpus", int),
                 ("steps", int), ("warmup", int), ("ms_per_step", float),
                 ("higher_is_better", bool), ("scaling", str), ("dtype", str), ("data", str),
                 ("config", dict), ("e2e", dict), ("roofline", dict), ("clocks", dict),
                 ("gpu_launches", int)):
        assert isinstance(d.get(k), t), (k, d.get(k))
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and abs(d["value"] - 1000.0 / d["ms_per_step"]) < 1e-6 * d["value"]
    assert "workload" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 1024 * 1024 * 3 and e["d2h_bytes_per_step"] == 8
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac"):
        assert k in r, k
    assert 0 < r["frac"] < 1 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["gpu_launches"] >= 30 * d["steps"]  # ~36 launches per step, all ours
