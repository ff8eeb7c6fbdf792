"""The C-ABI library builds for sm_100a, loads, and exports every entry point
declared in include/isogs.h (no compute: runs without a GPU)."""

from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "isogs.h")


def declared_symbols() -> list[str]:
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(isg_\w+)\s*\(", src, re.M)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("isg_knn_mean_grid", "isg_rank_of", "isg_chain_train_ranked", "isg_preprocess", "isg_sort_u64", "isg_sort_depth", "isg_sort_u16", "isg_bin_emit16",
              "isg_tile_offsets16", "isg_bin_count", "isg_bin_emit",
              "isg_raster_fwd", "isg_loss_l1_dssim", "isg_raster_bwd", "isg_reduce_ordered",
              "isg_chain", "isg_adam", "isg_chain_adam", "isg_raycast", "isg_iso_edges",
              "isg_iso_edge_points", "isg_iso_normals"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2509_05216_b200 import _lib as L
    lib = L.lib()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert L.SIGNATURES.keys() >= set(declared_symbols())
    assert b"sm_100a" in lib.isg_version()


def test_library_is_sm100a_only():
    from paper_2509_05216_b200 import _lib as L
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", L.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for other in ("sm_80", "sm_90"):
        assert other not in out


def test_entry_points_reject_bad_arguments_without_gpu():
    """Argument validation happens before any CUDA call."""
    from paper_2509_05216_b200 import _lib as L
    lib = L.lib()
    assert lib.isg_preprocess(None, None, 16, None, None) == 1  # cudaErrorInvalidValue
    assert lib.isg_sort_u64(None, None, None, None, None, None, -1, 0, 64, None) == 1
    assert lib.isg_adam(7, 1, None, None, None, None, None, None) == 1
    sz = ctypes.c_size_t(0)
    assert lib.isg_loss_l1_dssim(None, ctypes.byref(sz), 0, 5, 5, None, None, 0, 0.2, None, None, None) == 1
    dims = (ctypes.c_int32 * 3)(4, 4, 4)
    assert lib.isg_iso_edges(None, ctypes.byref(sz), None, ctypes.cast(dims, ctypes.c_void_p),
                             0, 2, 0.0, None, None, None) == 1  # stride 0
    assert lib.isg_raycast(None, None, None, None, 0.0, None, 0.5, 8, None, None, None, None,
                           None) == 1
