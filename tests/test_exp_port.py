"""The glibc-exact exp of csrc/glibc_exp.cuh reproduces the host libm exp
(what numba's np.exp calls on the key path) bit for bit.  Compiled for the
host with g++ here; the same header runs on the B200 (tests/test_parity_gpu.py)."""

from __future__ import annotations

import ctypes
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2509_05216_b200", "csrc")

HARNESS = r"""
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include "glibc_exp.cuh"
extern "C" long long mismatches(long long n, unsigned seed, double lo, double hi) {
    std::mt19937_64 g(seed);
    std::uniform_real_distribution<double> d(lo, hi);
    long long bad = 0;
    for (long long i = 0; i < n; i++) {
        double x = d(g);
        double a = isg::exp_glibc(x), b = std::exp(x);
        uint64_t ua, ub; std::memcpy(&ua, &a, 8); std::memcpy(&ub, &b, 8);
        bad += ua != ub;
    }
    return bad;
}
extern "C" double one(double x) { return isg::exp_glibc(x); }
"""


def _build(tmp_path):
    src = tmp_path / "h.cpp"
    src.write_text(HARNESS)
    so = tmp_path / "h.so"
    subprocess.run(["/usr/bin/g++", "-O2", "-mfma", "-ffp-contract=off", "-shared", "-fPIC",
                    "-I" + CSRC, str(src), "-o", str(so)], check=True)
    lib = ctypes.CDLL(str(so))
    lib.mismatches.restype = ctypes.c_longlong
    lib.mismatches.argtypes = [ctypes.c_longlong, ctypes.c_uint, ctypes.c_double, ctypes.c_double]
    lib.one.restype = ctypes.c_double
    lib.one.argtypes = [ctypes.c_double]
    return lib


def test_exp_port_matches_libm(tmp_path):
    lib = _build(tmp_path)
    # key-path ranges (2*log-scale, -logit), the raster range (power <= 0),
    # and the special-case ranges (|x| > 512, subnormal results)
    for lo, hi in ((-40.0, 10.0), (-6.0, 0.0), (-1e-3, 1e-3), (-745.0, -700.0),
                   (-800.0, 800.0), (500.0, 709.0)):
        assert lib.mismatches(400_000, 7, lo, hi) == 0, (lo, hi)


def test_exp_port_special_values(tmp_path):
    import math
    lib = _build(tmp_path)
    for x in (0.0, -0.0, 1e-300, -1e-300, 709.78, -745.2, -746.0, 710.0, 1.0, -1.0):
        assert lib.one(x) == math.exp(x) if x < 709.79 else math.isinf(lib.one(x))
    assert lib.one(float("-inf")) == 0.0
