"""ctypes binding of libisogs.so (include/isogs.h).

The package's only compute path.  Loading fails loudly -- there is no CPU or
PyTorch fallback: without the CUDA library or a CUDA device every op raises.
"""

from __future__ import annotations

import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ISOGS_LIB") or os.path.join(HERE, "_build", "libisogs.so")

ISG_F32 = 0
ISG_F64 = 1
TILE = 16

_lib = None


class IsgError(RuntimeError):
    """A libisogs entry point returned a CUDA error code."""


class Camera_t(ctypes.Structure):
    _fields_ = [("R", ctypes.c_double * 9), ("t", ctypes.c_double * 3),
                ("C", ctypes.c_double * 3), ("fx", ctypes.c_double), ("fy", ctypes.c_double),
                ("cx", ctypes.c_double), ("cy", ctypes.c_double), ("width", ctypes.c_int32),
                ("height", ctypes.c_int32)]


class Params_t(ctypes.Structure):
    _fields_ = [("positions", ctypes.c_void_p), ("log_scales", ctypes.c_void_p),
                ("rotations", ctypes.c_void_p), ("opacity_logits", ctypes.c_void_p),
                ("sh", ctypes.c_void_p), ("n", ctypes.c_int64), ("degree", ctypes.c_int32),
                ("dtype", ctypes.c_int32)]


class PreprocessOut_t(ctypes.Structure):
    _fields_ = [("key", ctypes.c_void_p), ("rect", ctypes.c_void_p), ("feat", ctypes.c_void_p),
                ("flag", ctypes.c_void_p), ("full64", ctypes.c_void_p),
                ("feat_dtype", ctypes.c_int32)]


class AdamConsts_t(ctypes.Structure):
    _fields_ = [(k, ctypes.c_double) for k in ("b1", "omb1", "b2", "omb2", "bc1", "bc2", "lr", "eps")]


class Chunks_t(ctypes.Structure):
    """isg_chunks (isogs.h): backward list chunking of the masked raster pair."""
    _fields_ = [("chunk", ctypes.c_int32), ("state", ctypes.c_void_p),
                ("items", ctypes.c_void_p), ("n_items", ctypes.c_void_p),
                ("max_items", ctypes.c_int32), ("image", ctypes.c_void_p),
                ("tile_last", ctypes.c_void_p), ("unroll2", ctypes.c_int32)]


class TrainState_t(ctypes.Structure):
    _fields_ = ([(k, ctypes.c_void_p) for k in (
        "positions", "log_scales", "rotations", "opacity_logits", "sh",
        "m_positions", "m_log_scales", "m_rotations", "m_opacity_logits", "m_sh",
        "v_positions", "v_log_scales", "v_rotations", "v_opacity_logits", "v_sh",
        "seen", "grad_accum")] + [("n", ctypes.c_int64), ("degree", ctypes.c_int32)])


# name -> argtypes (restype is int unless noted)
_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_D = ctypes.c_double
_SZ = ctypes.POINTER(ctypes.c_size_t)
SIGNATURES = {
    "isg_preprocess": [ctypes.POINTER(Params_t), ctypes.POINTER(Camera_t), _I32,
                       ctypes.POINTER(PreprocessOut_t), _P],
    "isg_sort_u64": [_P, _SZ, _P, _P, _P, _P, _I64, _I32, _I32, _P],
    "isg_sort_u32": [_P, _SZ, _P, _P, _P, _P, _I64, _I32, _I32, _P],
    "isg_sort_depth": [_P, _SZ, _P, _P, _P, _P, _I64, _P],
    "isg_bin_count_rows": [_P, _SZ, _I64, _P, _P, _P, _I32, _I32, _P, _P, _P, _P, _P],
    "isg_bin_count": [_P, _SZ, _I64, _P, _P, _P, _P, _I32, _I32, _I32, _P, _P, _P, _P, _P],
    "isg_bin_emit": [_I64, _P, _P, _I32, _I32, _I32, _P, _P, _P],
    "isg_rank_of": [_I64, _P, _P, _P, _P],
    "isg_tile_offsets": [_I64, _P, _I32, _P, _P],
    "isg_bin_emit16": [_I64, _P, _P, _I32, _I32, _I32, _P, _P, _P],
    "isg_sort_u16": [_P, _SZ, _P, _P, _P, _P, _I64, _I32, _I32, _P],
    "isg_tile_offsets16": [_I64, _P, _I32, _P, _P],
    "isg_raster_fwd": [_I32, _I32, _I32, _I32, _I32, _I32, _P, _I32, _P, _P, _P, _P, _P, _I32,
                       _P, _P, _P, _P, _P, _P],
    "isg_raster_fwd_masked": [_I32, _I32, _I32, _I32, _I32, _P, _I32, _P, _P, _P, _P, _P, _P,
                              _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "isg_raster_bwd_masked": [_I32, _I32, _I32, _I32, _I32, _P, _I32, _P, _P, _P, _P, _P, _P,
                              _P, _P, _P, _P, _I32, _P, _P, _P, _P, _P],
    "isg_bin_count_live": [_P, _SZ, _I64, _P, _P, _P, _P, _P, _I32, _I32, _P, _P, _P, _P, _P,
                           _P, _P],
    "isg_bin_emit_live": [_I64, _P, _P, _P, _P, _P, _I32, _I32, _I32, _P, _I32, _P, _P],
    "isg_chunk_state_floats": [_I64, _I32, _I32],
    "isg_chunk_items_max": [_I64, _I32, _I32],
    "isg_chunk_items": [_I32, _P, _P, _P, _I32, _I32, _P, _P, _P],
    "isg_tile_order_keys": [_I32, _P, _I32, _P, _P, _P],
    "isg_tile_order": [_I32, _P, _P, _P],
    "isg_sort_pairs_dev": [_P, _SZ, _I32, _P, _P, _P, _P, _I64, _P, _I32, _I32, _P],
    "isg_tile_offsets_dev": [_I64, _P, _P, _I32, _I32, _P, _P],
    "isg_contrib_mask_words": [_I64, _I32],
    "isg_loss_l1_dssim": [_P, _SZ, _I32, _I32, _I32, _P, _P, _I32, _D, _P, _P, _P],
    "isg_ssim": [_P, _SZ, _I32, _I32, _I32, _P, _P, _P, _P],
    "isg_raster_bwd": [_I32, _I32, _I32, _I32, _I32, _I32, _P, _I32, _P, _P, _P, _P, _P, _P,
                       _P, _P, _P, _I32, _P, _P],
    "isg_reduce_ordered": [_I32, _I64, _P, _P, _P, _P, _I32, _I32, _I32, _P, _P, _P],
    "isg_loss_partials_size": [_I32, _I32, _P, _P],
    "isg_loss_rows": [_P, _SZ, _I32, _I32, _I32, _I32, _I32, _P, _I32, _P, _I32, _D, _P, _P, _P,
                      _P],
    "isg_loss_finish": [_I32, _I32, _D, _P, _P, _P, _P],
    "isg_scan_i64": [_P, _SZ, _I64, _P, _P, _P, _P],
    "isg_route_plan_size": [_I64, _I32, _P],
    "isg_route_plan": [_I64, _P, _P, _P, _I32, _I32, _P, _P, _P],
    "isg_route_pack": [_I64, _P, _P, _P, _P, _P, _I32, _P, _P, _I32, _P, _P, _P, _P, _P],
    "isg_route_mask": [_I64, _P, _I32, _I32, _P, _P],
    "isg_band_blocks": [_I64, _P, _I32, _I32, _I32, _P, _P],
    "isg_band_fold": [_I64, _P, _P, _P, _P, _P, _I32, _I32, _I32, _I32, _P, _P],
    "isg_band_fold_peer": [_I64, _P, _P, _P, _P, _P, _I32, _I32, _I32, _I32, _I32, _P, _P, _P],
    "isg_route_pack_peer": [_I64, _P, _P, _P, _P, _P, _I32, _P, _P, _P, _P],
    "isg_copy": [_P, _P, _I64, _P],
    "isg_preprocess_devcam": [ctypes.POINTER(Params_t), _P, _I32, _I32, _I32,
                              ctypes.POINTER(PreprocessOut_t), _P],
    "isg_bin_count_train": [_P, _SZ, _I64, _P, _P, _P, _P, _I32, _I32, _P, _P, _P, _P, _P, _P,
                            _P],
    "isg_compact_count": [_P, _SZ, _I64, _P, _P, _P],
    "isg_compact_batch": [_I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "isg_gather_batch": [_I64, _P, _P, _P, _P, _P, _P, _P, _I32, _P, _P, _P],
    "isg_densify_classify": [_I64, _P, _P, _P, _P, _D, _D, _I32, _D, _D, _P, _P],
    "isg_reduce_live": [_I64, _P, _P, _P, _P, _I32, _I32, _I32, _P, _P, _P],
    "isg_band_cost": [_P, _I32, _I32, _I32, _I32, _P, _P],
    "isg_owner_fold_plan": [_I64, _P, _P, _P, _I32, _I32, _P, _P, _P, _P],
    "isg_grad_rows": [_I64, _P, _P, _P, _P],
    "isg_owner_fold": [_I64, _P, _P, _P, _P, _P],
    "isg_chain": [ctypes.POINTER(Params_t), ctypes.POINTER(Camera_t), _P, _P, _P, _P, _P, _P,
                  _P, _P],
    "isg_adam": [_I32, _I64, _P, _P, _P, _P, ctypes.POINTER(AdamConsts_t), _P],
    "isg_chain_adam": [ctypes.POINTER(TrainState_t), ctypes.POINTER(Camera_t), _P, _P, _P,
                       ctypes.POINTER(AdamConsts_t), _D, _D, _P],
    "isg_chain_fold_adam": [ctypes.POINTER(TrainState_t), ctypes.POINTER(Camera_t), _P, _P, _P,
                            _P, _I32, _I32, _I32, _P, _P, _P, ctypes.POINTER(AdamConsts_t), _D,
                            _D, _P],
    "isg_chain_adam_train": [ctypes.POINTER(TrainState_t), ctypes.POINTER(Camera_t), _P, _P, _P,
                             _P, ctypes.POINTER(AdamConsts_t), _D, _D, _P],
    "isg_chain_train": [ctypes.POINTER(Params_t), ctypes.POINTER(Camera_t), _P, _P, _P, _P, _P,
                        _P, _P, _P, _P, _D, _D, _P],
    "isg_chain_train_ranked": [ctypes.POINTER(Params_t), ctypes.POINTER(Camera_t), _P, _P, _P,
                               _P, _P, _P, _P, _P, _P, _D, _D, _P],
    "isg_chain_fold_train": [ctypes.POINTER(Params_t), ctypes.POINTER(Camera_t), _P, _P, _P, _P,
                             _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _D, _D, _P],
    "isg_adam_groups": [_I32, _P, _P, _P, _P, _P, _P, ctypes.POINTER(AdamConsts_t), _P],
    "isg_exp_f64": [_I64, _P, _P, _P],
    "isg_probe_ffma": [_I32, _I32, _P, _P],
    "isg_knn_mean_grid": [_P, _SZ, _P, _I64, _I32, _P, _D, _I64, _I64, _I64, _P, _P],
    "isg_raycast": [_P, _P, _P, _P, _D, ctypes.POINTER(Camera_t), _D, _I32, _P, _P, _P, _P, _P],
    "isg_iso_edges": [_P, _SZ, _P, _P, _I32, _I32, _D, _P, _P, _P],
    "isg_iso_edge_points": [_P, _P, _P, _P, _I32, _I32, _D, _I64, _P, _P, _P],
    "isg_iso_normals": [_P, _P, _P, _P, _I64, _P, _P, _P],
    "isg_version": [],
}


RET_I64 = ("isg_contrib_mask_words", "isg_chunk_state_floats")


def lib():
    """Load libisogs.so (building it first if the sources are newer)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            from . import build as _build
            _build.build()
        L = ctypes.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = (ctypes.c_char_p if name == "isg_version" else
                          ctypes.c_int64 if name in RET_I64 else ctypes.c_int)
        _lib = L
    return _lib


def check(code: int, what: str) -> None:
    if code != 0:
        raise IsgError(f"{what} failed with CUDA error {code}")


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2509_05216_b200 needs a CUDA device (B200); "
                           "there is no CPU fallback")
    lib()
    return torch.device("cuda", torch.cuda.current_device())


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    return t.data_ptr()


def stream_ptr() -> int:
    # the current stream's raw handle straight from the C++ side (a
    # torch.cuda.current_stream() object costs ~15 us of Python per call)
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


def dtype_tag(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return ISG_F32
    if dt == torch.float64:
        return ISG_F64
    raise ValueError(f"unsupported dtype {dt}")


def camera_struct(cam) -> Camera_t:
    import numpy as np
    c = Camera_t()
    r = np.asarray(cam.rotation, dtype=np.float64).reshape(3, 3)
    t = np.asarray(cam.translation, dtype=np.float64).reshape(3)
    pos = -r.T @ t
    for i in range(9):
        c.R[i] = float(r.reshape(9)[i])
    for i in range(3):
        c.t[i] = float(t[i])
        c.C[i] = float(pos[i])
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.width, c.height = int(cam.width), int(cam.height)
    return c


class Workspace:
    """Grow-only device scratch buffer for the two-phase workspace queries."""

    def __init__(self):
        self.buf: torch.Tensor | None = None

    def get(self, nbytes: int, device) -> torch.Tensor:
        nbytes = max(int(nbytes), 1)
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != device:
            self.buf = torch.empty(int(nbytes * 1.25) + 256, dtype=torch.uint8, device=device)
        return self.buf


def sort_depth(keys: torch.Tensor, vals: torch.Tensor, ws: Workspace,
               keys_out: torch.Tensor | None = None, vals_out: torch.Tensor | None = None):
    """The global depth order: stable sort of (float64 depth bits, id) pairs
    (isg_sort_depth; identical to a full 64-bit sort_pairs)."""
    n = keys.numel()
    if keys_out is None:
        keys_out = torch.empty_like(keys)
    if vals_out is None:
        vals_out = torch.empty_like(vals)
    if n == 0:
        return keys_out, vals_out
    L = lib()
    sz = ctypes.c_size_t(0)
    check(L.isg_sort_depth(None, ctypes.byref(sz), ptr(keys), ptr(keys_out), ptr(vals),
                           ptr(vals_out), n, None), "sort_depth (size query)")
    buf = ws.get(sz.value, keys.device)
    sz = ctypes.c_size_t(buf.numel())
    check(L.isg_sort_depth(ptr(buf), ctypes.byref(sz), ptr(keys), ptr(keys_out), ptr(vals),
                           ptr(vals_out), n, stream_ptr()), "sort_depth")
    return keys_out, vals_out


def sort_pairs(keys: torch.Tensor, vals: torch.Tensor, bits: tuple[int, int],
               ws: Workspace, keys_out: torch.Tensor | None = None,
               vals_out: torch.Tensor | None = None):
    """Stable radix sort of (uint key, int32 value) pairs (isg_sort_u64/u32)."""
    n = keys.numel()
    if keys_out is None:
        keys_out = torch.empty_like(keys)
    if vals_out is None:
        vals_out = torch.empty_like(vals)
    if n == 0:
        return keys_out, vals_out
    L = lib()
    fn = {8: L.isg_sort_u64, 4: L.isg_sort_u32, 2: L.isg_sort_u16}[keys.element_size()]
    sz = ctypes.c_size_t(0)
    check(fn(None, ctypes.byref(sz), ptr(keys), ptr(keys_out), ptr(vals), ptr(vals_out), n,
             bits[0], bits[1], None), "sort (size query)")
    buf = ws.get(sz.value, keys.device)
    sz = ctypes.c_size_t(buf.numel())
    check(fn(ptr(buf), ctypes.byref(sz), ptr(keys), ptr(keys_out), ptr(vals), ptr(vals_out), n,
             bits[0], bits[1], stream_ptr()), "sort")
    return keys_out, vals_out
