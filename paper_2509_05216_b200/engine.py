"""Device-resident training step (reference engine.py:465-562) on one B200.

One iteration is a fixed chain of libisogs launches on the current stream:

  isg_preprocess   project every Gaussian (fp64 key path)        N rows
  isg_sort_depth   global (depth, id) order (hand-written radix)   N keys
  isg_bin_count    rank-order gather + tile-count scan             N ranks
  [D2H 16 B]       M visible, E tile entries (sizes the E buffers)
  isg_bin_emit     (tile, rank) pairs in rank order                E pairs
  isg_sort_u32     stable sort on tile id -> per-tile lists        E pairs
  isg_tile_offsets CSR offsets                                     T tiles
  isg_raster_fwd   front-to-back composite                         P pixels
  isg_loss_l1_dssim fused L1 + D-SSIM and dL/dimage                P pixels
  isg_raster_bwd   per-(tile, splat) subtotals                     P pixels
  isg_reduce_ordered ascending-tile fold per splat (fp64)          M ranks
  isg_chain_adam   chain rule + stats + dense Adam                 N rows

The only host synchronisation is the 16-byte read of (M, E).  Buffers are
capacity-managed and reused across iterations; nothing is allocated in the
steady state.  W > 1 lives in distributed.py.
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .gaussians import PARAM_NAMES, GaussianCloud, cloud_from_points, to_device_cloud
from .metrics import loss_l1_dssim_device, psnr, quantize8, ssim
from .optim import adam_consts, position_lr
from .training import (EvalRecord, TrainConfig, TrainDataset, TrainReport, TrainStats,
                       build_schedule, init_log_scales)

TILE = 16
# Canonical fold grouping (tile rows per block): every per-splat gradient is
# summed tiles-ascending inside 2-tile-row blocks, then block sums ascending.
# Pixel bands of the multi-GPU step are unions of whole blocks, which makes
# the result bitwise independent of the GPU count (see csrc/dist.cu).  Two
# rows: bands can be cut at 32-pixel granularity for load balance
# (tools/band_balance.py: 8 rows leave 1.26-1.30 max/mean at W=8) for ~1.7
# gradient records per splat instead of ~1.2.
CANON_ROWS = 2


def _iota(buf: torch.Tensor | None, n: int, device) -> torch.Tensor:
    """0, 1, 2, ... of at least n entries (int32), grown on demand."""
    if buf is None or buf.shape[0] < n:
        return torch.arange(max(int(n * 1.25), 16), dtype=torch.int32, device=device)
    return buf


def _grow(buf: torch.Tensor | None, n: int, shape_tail=(), dtype=torch.float32, device=None,
          slack: float = 1.25) -> torch.Tensor:
    if buf is None or buf.shape[0] < n:
        cap = max(int(n * slack), 16)
        return torch.empty((cap,) + tuple(shape_tail), dtype=dtype, device=device)
    return buf


class PhaseTimer:
    """CUDA events between launches on the current stream: phase name ->
    device milliseconds (used by bench.py for the per-kernel roofline)."""

    def __init__(self):
        self.marks: list[tuple[str, torch.cuda.Event]] = []

    def mark(self, name: str) -> None:
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.marks.append((name, e))

    def phases(self) -> dict[str, float]:
        torch.cuda.synchronize()
        out: dict[str, float] = {}
        for (_, a), (name, b) in zip(self.marks[:-1], self.marks[1:]):
            out[name] = out.get(name, 0.0) + a.elapsed_time(b)
        return out


def _mark(timer, name):
    if timer is not None:
        timer.mark(name)


@dataclass
class ViewContext:
    """Per-view forward state kept for the backward (the cache of RenderAux)."""

    m: int
    e: int          # tile-list entries
    slots: int = 0  # subtotal slots (= e unless the lists are live-only)


class Rasterizer:
    """Buffers + launch sequence for one view on one GPU (band = all rows)."""

    def __init__(self, n: int, width: int, height: int, device, background=(1.0, 1.0, 1.0),
                 feat_dtype=torch.float32, canon_rows: int = CANON_ROWS):
        self.canon_rows = canon_rows
        self.device = device
        self.width, self.height = width, height
        self.tiles_x = (width + TILE - 1) // TILE
        self.tiles_y = (height + TILE - 1) // TILE
        self.n_tiles = self.tiles_x * self.tiles_y
        self.image_tiles = self.n_tiles  # (the chunk policy's input)
        self.tile_bits = max(1, int(self.n_tiles - 1).bit_length())
        self.bg = (ctypes.c_double * 3)(*[float(v) for v in background])
        self.feat_dtype = feat_dtype
        self.ftag = L.dtype_tag(feat_dtype)
        self.ws_sort = L.Workspace()
        self.ws_bin = L.Workspace()
        self.counts_host = torch.zeros(3, dtype=torch.int64).pin_memory()
        self.resize(n)
        dev = device
        self.image = torch.empty((height, width, 3), dtype=torch.float32, device=dev)
        self.t_final = torch.empty((height, width), dtype=feat_dtype, device=dev)
        self.n_last = torch.empty((height, width), dtype=torch.int32, device=dev)
        self.dl = torch.empty((height, width, 3), dtype=torch.float32, device=dev)
        self.offsets = torch.empty(self.n_tiles + 1, dtype=torch.int32, device=dev)
        self.tile_keys = self.tile_vals = self.keys_sorted_t = self.entries = None
        self.slot_rank = self.iota = None
        self.live = False  # live-only training lists (isg_bin_emit_live)
        # the training step folds the live subtotals inside the chain kernel
        # (ranked grads only); keep_grad2d also stores the 2-D gradients
        self.fuse_fold = os.environ.get("ISOGS_FUSE_FOLD", "1") != "0"
        self.keep_grad2d = False
        self.keep_grads = False  # store the parameter gradients (fused Adam)
        self.graph = self.graph_key = None  # the captured pre-sync launches
        self.partials = None
        self.to_keys = self.to_vals = self.to_keys_s = self.to_order = None
        self.tile_order = None
        self.chunks = None
        self.chunk = CHUNK  # backward entries per work item (0: one CTA per tile; None: auto)
        # launch the raster pair heaviest tile lists first (ISOGS_HEAVY_FIRST=0: list order)
        self.heavy_first = os.environ.get("ISOGS_HEAVY_FIRST", "1") != "0"
        # float32: forward contribution masks drive the backward (ISOGS_CMASK=0: A/B off)
        self.use_cmask = os.environ.get("ISOGS_CMASK", "1") != "0"
        self.cmask = None
        self.cmask_ok = False
        self.n_contrib_out = None  # set to (H, W) int32 tensors to count pairs
        self.n_iter_out = None
        self.timer: PhaseTimer | None = None
        # training step: grad2d in rank order (coalesced fold output), read by
        # the chain through rank_of (isg_chain_train_ranked)
        self.ranked_grads = False

    def resize(self, n: int) -> None:
        dev = self.device
        self.n = n
        self.key = torch.empty(n, dtype=torch.int64, device=dev)
        self.rect = torch.empty((n, 4), dtype=torch.int32, device=dev)
        self.feat = torch.empty((n, 12), dtype=self.feat_dtype, device=dev)
        self.flag = torch.empty(n, dtype=torch.uint8, device=dev)
        self.vals0 = torch.arange(n, dtype=torch.int32, device=dev)
        self.key_sorted = torch.empty(n, dtype=torch.int64, device=dev)
        self.order = torch.empty(n, dtype=torch.int32, device=dev)
        self.rect_sorted = torch.empty((n, 4), dtype=torch.int32, device=dev)
        self.feat_sorted = torch.empty((n, 12), dtype=self.feat_dtype, device=dev)
        self.emit_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
        self.rank_of = torch.empty(n, dtype=torch.int32, device=dev)
        self.live_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
        self.live_mask = torch.empty(n, dtype=torch.int64, device=dev)
        self.counts = torch.zeros(3, dtype=torch.int64, device=dev)
        self.grad2d = torch.empty((n, 9), dtype=torch.float64, device=dev)

    def _presync(self, p, out, live: bool, n: int, tm, cam_dev=None) -> None:
        """The step's launches before its one host read: preprocess, depth
        sort, binning (live counts, the rank inverse)."""
        lib = L.lib()
        s = L.stream_ptr()
        if cam_dev is not None:
            L.check(lib.isg_preprocess_devcam(ctypes.byref(p), L.ptr(cam_dev), self.width,
                                              self.height, TILE, ctypes.byref(out), s),
                    "isg_preprocess_devcam")
        else:
            L.check(lib.isg_preprocess(ctypes.byref(p), ctypes.byref(self.cam_struct), TILE,
                                       ctypes.byref(out), s), "isg_preprocess")
        _mark(tm, "preprocess")
        L.sort_depth(self.key, self.vals0, self.ws_sort, self.key_sorted, self.order)
        _mark(tm, "sort_depth")
        sz = ctypes.c_size_t(0)
        if live:
            L.check(lib.isg_bin_count_train(None, ctypes.byref(sz), n, None, None, None, None, 0,
                                            self.tiles_y, None, None, None, None, None, None,
                                            None), "bin (size)")
        else:
            L.check(lib.isg_bin_count(None, ctypes.byref(sz), n, None, None, None, None,
                                      self.ftag, 0, self.tiles_y, None, None, None, None, None),
                    "bin (size)")
        ws = self.ws_bin.get(sz.value, self.device)
        sz = ctypes.c_size_t(ws.numel())
        if live:
            # live lists only (no full-layout offsets), the rank inverse fused
            L.check(lib.isg_bin_count_train(L.ptr(ws), ctypes.byref(sz), n,
                                            L.ptr(self.key_sorted), L.ptr(self.order),
                                            L.ptr(self.rect), L.ptr(self.feat), 0, self.tiles_y,
                                            L.ptr(self.rect_sorted), L.ptr(self.feat_sorted),
                                            L.ptr(self.live_off), L.ptr(self.live_mask),
                                            L.ptr(self.rank_of) if self.ranked_grads else None,
                                            L.ptr(self.counts), s), "isg_bin_count_train")
        else:
            L.check(lib.isg_bin_count(L.ptr(ws), ctypes.byref(sz), n, L.ptr(self.key_sorted),
                                      L.ptr(self.order), L.ptr(self.rect), L.ptr(self.feat),
                                      self.ftag, 0, self.tiles_y, L.ptr(self.rect_sorted),
                                      L.ptr(self.feat_sorted), L.ptr(self.emit_off),
                                      L.ptr(self.counts), s), "isg_bin_count")
        if self.ranked_grads and not live:
            L.check(lib.isg_rank_of(n, L.ptr(self.key_sorted), L.ptr(self.order),
                                    L.ptr(self.rank_of), s), "isg_rank_of")

    def _presync_graph(self, cloud, p, out) -> None:
        """_presync as one CUDA graph replay: the launches depend only on the
        Gaussian count and the buffers, the camera is uploaded to device
        memory before each replay.  Captured after one eager run (which
        sizes every workspace) and re-captured when the cloud changes."""
        n = cloud.count
        key = (n, cloud.degree, L.ptr(cloud.positions), L.ptr(cloud.log_scales),
               L.ptr(cloud.rotations), L.ptr(cloud.opacity_logits), L.ptr(cloud.sh_coeffs),
               L.ptr(self.key), self.ranked_grads)
        nb = ctypes.sizeof(L.Camera_t)
        if getattr(self, "cam_dev", None) is None:
            self.cam_dev = torch.empty(nb, dtype=torch.uint8, device=self.device)
            self.cam_pin = torch.empty(nb, dtype=torch.uint8).pin_memory()
        ctypes.memmove(self.cam_pin.data_ptr(), ctypes.addressof(self.cam_struct), nb)
        self.cam_dev.copy_(self.cam_pin, non_blocking=True)
        if self.graph is not None and self.graph_key == key:
            self.graph.replay()
            return
        # eager run for this step (sizes the workspaces), then capture
        self._presync(p, out, True, n, None, self.cam_dev)
        self.graph = None
        g = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            self._presync(p, out, True, n, None, self.cam_dev)
        self.graph, self.graph_key = g, key

    # -- forward ---------------------------------------------------------
    def forward(self, cloud: GaussianCloud, cam) -> ViewContext:
        lib = L.lib()
        s = L.stream_ptr()
        n = cloud.count
        if n != self.n:
            self.resize(n)
        out = L.PreprocessOut_t()
        out.key, out.rect, out.feat = L.ptr(self.key), L.ptr(self.rect), L.ptr(self.feat)
        out.flag, out.full64, out.feat_dtype = L.ptr(self.flag), None, self.ftag
        p = L.Params_t()
        p.positions, p.log_scales = L.ptr(cloud.positions), L.ptr(cloud.log_scales)
        p.rotations, p.opacity_logits = L.ptr(cloud.rotations), L.ptr(cloud.opacity_logits)
        p.sh, p.n, p.degree, p.dtype = L.ptr(cloud.sh_coeffs), n, cloud.degree, L.ISG_F32
        self.cam_struct = L.camera_struct(cam)
        tm = self.timer
        _mark(tm, "begin")
        # float32 training lists are live-only: a (tile, splat) pair no pixel of
        # the tile can composite has no list entry and no subtotal slot
        live = self.use_cmask and self.feat_dtype == torch.float32
        self.live = live
        if GRAPH and live and tm is None and n:
            self._presync_graph(cloud, p, out)
        else:
            self._presync(p, out, live, n, tm)
        _mark(tm, "bin_count")
        self.counts_host.copy_(self.counts, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        _mark(tm, "host_sync")
        m, e_full = int(self.counts_host[0]), int(self.counts_host[1])
        e = int(self.counts_host[2]) if live else e_full
        dev = self.device
        k16 = self.n_tiles <= 65536  # 2-byte tile keys: less sort traffic
        kdt = torch.int16 if k16 else torch.int32
        if self.tile_keys is None or self.tile_keys.dtype != kdt:
            self.tile_keys = self.keys_sorted_t = None
        self.tile_keys = _grow(self.tile_keys, e, dtype=kdt, device=dev)
        self.tile_vals = _grow(self.tile_vals, e, dtype=torch.int32, device=dev)
        self.keys_sorted_t = _grow(self.keys_sorted_t, e, dtype=kdt, device=dev)
        self.entries = _grow(self.entries, e, dtype=torch.int32, device=dev)
        offs = lib.isg_tile_offsets16 if k16 else lib.isg_tile_offsets
        if e:
            if live:
                self.slot_rank = _grow(self.slot_rank, e, dtype=torch.int32, device=dev)
                L.check(lib.isg_bin_emit_live(m, L.ptr(self.rect_sorted), L.ptr(self.emit_off),
                                              L.ptr(self.live_off), L.ptr(self.live_mask),
                                              L.ptr(self.feat_sorted), self.tiles_x, 0,
                                              self.tiles_y, L.ptr(self.tile_keys),
                                              2 if k16 else 4, L.ptr(self.slot_rank), s),
                        "isg_bin_emit_live")
                # the sort's values are the slots themselves: 0..e-1
                self.iota = _iota(self.iota, e, dev)
                vals = self.iota
            else:
                emit = lib.isg_bin_emit16 if k16 else lib.isg_bin_emit
                L.check(emit(m, L.ptr(self.rect_sorted), L.ptr(self.emit_off), self.tiles_x, 0,
                             self.tiles_y, L.ptr(self.tile_keys), L.ptr(self.tile_vals), s),
                        "isg_bin_emit")
                vals = self.tile_vals
            _mark(tm, "bin_emit")
            L.sort_pairs(self.tile_keys[:e], vals[:e], (0, self.tile_bits),
                         self.ws_sort, self.keys_sorted_t[:e], self.entries[:e])
            _mark(tm, "sort_tiles")
        L.check(offs(e, L.ptr(self.keys_sorted_t), self.n_tiles, L.ptr(self.offsets), s),
                "isg_tile_offsets")
        self.tile_order = heavy_first_order(self, self.n_tiles, self.offsets)
        self.chunks = (chunk_setup(self, self.n_tiles, e, L.ptr(self.image))
                       if self.use_cmask and self.feat_dtype == torch.float32 else None)
        _mark(tm, "tile_offsets")
        self.cmask_ok = self.use_cmask and self.feat_dtype == torch.float32
        if self.cmask_ok:
            # the forward leaves per-(tile, quadrant, batch) contribution masks
            # that the backward walks instead of re-culling every entry
            words = lib.isg_contrib_mask_words(e, self.n_tiles)
            self.cmask = _grow(self.cmask, words, dtype=torch.int32, device=dev)
            L.check(lib.isg_raster_fwd_masked(
                self.width, self.height, self.tiles_x, 0, self.tiles_y, None, 0,
                L.ptr(self.tile_order),
                L.ptr(self.offsets), L.ptr(self.entries), L.ptr(self.feat_sorted),
                ctypes.cast(self.bg, ctypes.c_void_p), L.ptr(self.image), L.ISG_F32,
                L.ptr(self.t_final), L.ptr(self.n_last), L.ptr(self.n_contrib_out),
                L.ptr(self.n_iter_out), None, L.ptr(self.cmask),
                ctypes.byref(self.chunks) if self.chunks is not None else None,
                L.ptr(self.slot_rank) if self.live else None, s),
                "isg_raster_fwd_masked")
        else:
            L.check(lib.isg_raster_fwd(self.ftag, self.width, self.height, self.tiles_x, 0,
                                       self.tiles_y, None, 0, L.ptr(self.offsets),
                                       L.ptr(self.entries), L.ptr(self.feat_sorted),
                                       ctypes.cast(self.bg, ctypes.c_void_p), L.ptr(self.image),
                                       L.ISG_F32, L.ptr(self.t_final), L.ptr(self.n_last),
                                       L.ptr(self.n_contrib_out), L.ptr(self.n_iter_out), None,
                                       s), "isg_raster_fwd")
        _mark(tm, "raster_fwd")
        return ViewContext(m=m, e=e, slots=e)

    # -- backward --------------------------------------------------------
    def backward(self, ctx: ViewContext) -> None:
        lib = L.lib()
        s = L.stream_ptr()
        # float32 records are padded to 12 floats (isogs.h: isg_raster_bwd)
        rec = 12 if self.feat_dtype == torch.float32 else 9
        self.partials = _grow(self.partials, max(ctx.slots, ctx.e, 1), (rec,), dtype=self.feat_dtype,
                              device=self.device)
        if self.cmask_ok:
            chunk_items(self, self.n_tiles)
            L.check(lib.isg_raster_bwd_masked(
                self.width, self.height, self.tiles_x, 0, self.tiles_y, None, 0,
                L.ptr(self.tile_order),
                L.ptr(self.offsets), L.ptr(self.entries), L.ptr(self.feat_sorted),
                L.ptr(self.rect_sorted), L.ptr(self.emit_off),
                ctypes.cast(self.bg, ctypes.c_void_p), L.ptr(self.t_final), L.ptr(self.n_last),
                L.ptr(self.dl), L.ISG_F32, L.ptr(self.partials), L.ptr(self.cmask),
                ctypes.byref(self.chunks) if self.chunks is not None else None,
                L.ptr(self.slot_rank) if self.live else None, s),
                "isg_raster_bwd_masked")
        else:
            L.check(lib.isg_raster_bwd(self.ftag, self.width, self.height, self.tiles_x, 0,
                                       self.tiles_y, None, 0, L.ptr(self.offsets),
                                       L.ptr(self.entries), L.ptr(self.feat_sorted),
                                       L.ptr(self.rect_sorted), L.ptr(self.emit_off),
                                       ctypes.cast(self.bg, ctypes.c_void_p), L.ptr(self.t_final),
                                       L.ptr(self.n_last), L.ptr(self.dl), L.ISG_F32,
                                       L.ptr(self.partials), s), "isg_raster_bwd")
        _mark(self.timer, "raster_bwd")
        if ctx.m and self.live and self.fuse_fold and self.ranked_grads:
            pass  # folded inside the chain (isg_chain_fold_train)
        elif ctx.m and self.live:
            L.check(lib.isg_reduce_live(ctx.m, L.ptr(self.live_off), L.ptr(self.partials),
                                        None if self.ranked_grads else L.ptr(self.order),
                                        L.ptr(self.rect_sorted), 0, self.tiles_y,
                                        self.canon_rows, L.ptr(self.grad2d), None, s),
                    "isg_reduce_live")
        elif ctx.m:
            L.check(lib.isg_reduce_ordered(self.ftag, ctx.m, L.ptr(self.emit_off),
                                           L.ptr(self.partials),
                                           None if self.ranked_grads else L.ptr(self.order),
                                           L.ptr(self.rect_sorted), 0, self.tiles_y,
                                           self.canon_rows,
                                           L.ptr(self.grad2d), None, s), "isg_reduce_ordered")
        _mark(self.timer, "reduce")

    LAUNCHES_PER_STEP = None  # filled by Trainer (documented count)


# Tiles whose list is at least HEAVY_PCT % of the mean length launch first
# (longest first); the rest keep row-major order (0: all by length).
HEAVY_PCT = int(os.environ.get("ISOGS_HEAVY_PCT", "0"))
# the step's launches before its host read (preprocess, depth sort, binning)
# as one CUDA graph replay (ISOGS_GRAPH=0: eager launches)
GRAPH = os.environ.get("ISOGS_GRAPH", "1") != "0"
# chain rule + stats + Adam in one pass (the gradients stay in registers;
# isg_chain_fold_adam).  Off by default: measured slower at config 3 (1.14 ms
# against 0.63 + 0.39 ms for the fold-chain and the dense Adam launches) --
# the fused kernel's register footprint costs the latency-bound fold more
# occupancy than the 0.74 GB of gradient traffic it saves.
FUSE_ADAM = os.environ.get("ISOGS_FUSE_ADAM", "0") != "0"
# heavy-first launch order: one launch bucketing the tiles by list length
# (isg_tile_order, 1024 linear buckets; default) or the exact longest-first
# order (a 16-bit radix sort of the lengths, 8 launches for 16K keys):
# measured 119.0 -> 119.6 images/s at config 3, 469 -> 477 at config 2
EXACT_ORDER = os.environ.get("ISOGS_EXACT_ORDER", "0") != "0"


def heavy_first_order(st, n_tiles: int, offsets: torch.Tensor):
    """Launch order of the raster pair, heaviest tile lists first (one launch,
    isg_tile_order: tiles bucketed by list length; EXACT_ORDER / HEAVY_PCT:
    isg_tile_order_keys + a 16-bit stable sort): with one CTA per tile, a long
    list launched last runs alone at the end of the kernel; launched first it
    overlaps the light ones.  The order is the launch order only -- results
    do not depend on it.  `st` holds the scratch buffers and the heavy_first
    switch.  Returns None (list order) when off."""
    if not st.heavy_first or n_tiles < 2:
        return None
    lib = L.lib()
    dev = offsets.device
    st.to_order = _grow(st.to_order, n_tiles, dtype=torch.int32, device=dev)
    if HEAVY_PCT == 0 and not EXACT_ORDER:
        # one launch: tiles bucketed by list bit length, longest first
        L.check(lib.isg_tile_order(n_tiles, L.ptr(offsets), L.ptr(st.to_order), L.stream_ptr()),
                "isg_tile_order")
        return st.to_order
    st.to_keys = _grow(st.to_keys, n_tiles, dtype=torch.int16, device=dev)
    st.to_vals = _grow(st.to_vals, n_tiles, dtype=torch.int32, device=dev)
    st.to_keys_s = _grow(st.to_keys_s, n_tiles, dtype=torch.int16, device=dev)
    L.check(lib.isg_tile_order_keys(n_tiles, L.ptr(offsets), HEAVY_PCT, L.ptr(st.to_keys),
                                    L.ptr(st.to_vals), L.stream_ptr()), "isg_tile_order_keys")
    if not hasattr(st, "ws_order"):
        st.ws_order = L.Workspace()
    L.sort_pairs(st.to_keys[:n_tiles], st.to_vals[:n_tiles], (0, 16), st.ws_order,
                 st.to_keys_s[:n_tiles], st.to_order[:n_tiles])
    return st.to_order


# Backward list chunking: ISOGS_CHUNK=<entries> forces a chunk size (0: off).
# By default (auto) the chunk follows the IMAGE's tile count, never the
# launch's: images of few tiles (config 2: 4096 tiles, about 2 waves of
# backward CTAs, where one CTA per tile leaves the heaviest lists running
# alone at the end) are chunked, larger ones (2048^2) are not.  A function of
# the workload only, so every row band of every GPU count cuts the same
# chunks as one GPU and the sharded step stays bitwise equal to it (chunk
# restarts round differently from an unbroken walk).  Measured: config 2
# 416 -> 458 images/s at 1024; config 3 116.8 -> 107.1 (the chunked
# instantiation rematerialises lane indices under register pressure: +3.5 %
# instructions, 12 vs 14 CTAs/SM); emulated W = 8 config-3 bands would gain
# 410 -> 438 with per-band chunking, at the cost of that bitwise equality.
_ck = os.environ.get("ISOGS_CHUNK", "auto")
CHUNK = None if _ck == "auto" else int(_ck)
AUTO_CHUNK = 1024
AUTO_CHUNK_TILES = 6144


def chunk_size(image_tiles: int, forced=None) -> int:
    """The backward chunk for an image of `image_tiles` tiles (0: one CTA per
    tile list); `forced` (an int) overrides."""
    if forced is not None:
        return forced
    return AUTO_CHUNK if 0 < image_tiles <= AUTO_CHUNK_TILES else 0
SPLIT_TILES = 1 << 30  # every chunk its own CTA when chunking is on
# Unchunked backward launches of at most UNROLL2_TILES lists take three entries
# per step (bwd_kernel<..., 3>: the same bits, more instruction-level
# parallelism for the heaviest lists that finish alone on their SMs; a
# per-launch choice, so any band split keeps its results).
# Measured (emulated config-3 ranks): W = 8 bands of 2048 lists 470 -> 490
# images/s; W = 4 bands of 4096 lists 311 -> 305; one GPU (16384 lists) 126 ->
# 115.  Default: launches of at most 2560 lists.
_u2 = os.environ.get("ISOGS_BWD_UNROLL2", "2560")
UNROLL2_TILES = 0 if _u2 == "0" else (1 << 30 if _u2 == "1" else int(_u2))


def unroll2(n_tiles: int) -> bool:
    return 0 < n_tiles <= UNROLL2_TILES


def chunk_setup(st, n_tiles: int, e: int, image_ptr: int):
    """isg_chunks for the masked raster pair over `n_tiles` lists with `e`
    entries (the boundary-state and per-quadrant last-position buffers); the
    work items are built between the forward and the backward by
    chunk_items().  `st` holds the buffers.  None when off."""
    chunk = chunk_size(st.image_tiles, getattr(st, "chunk", CHUNK))
    if n_tiles == 0:
        return None
    if chunk <= 0:
        if not unroll2(n_tiles):
            return None
        c = L.Chunks_t()  # unchunked, two entries per backward step
        c.unroll2 = 1
        return c
    lib = L.lib()
    dev = st.offsets.device
    nst = int(lib.isg_chunk_state_floats(e, n_tiles, chunk))
    st.ch_state = _grow(getattr(st, "ch_state", None), nst, dtype=torch.float32, device=dev)
    mx = int(lib.isg_chunk_items_max(e, n_tiles, chunk))
    st.ch_items = _grow(getattr(st, "ch_items", None), 2 * mx, dtype=torch.int32, device=dev)
    st.ch_last = _grow(getattr(st, "ch_last", None), 4 * n_tiles, dtype=torch.int32, device=dev)
    if getattr(st, "ch_n", None) is None:
        st.ch_n = torch.zeros(1, dtype=torch.int32, device=dev)
    c = L.Chunks_t()
    c.chunk, c.state, c.items, c.n_items = chunk, L.ptr(st.ch_state), L.ptr(st.ch_items), L.ptr(st.ch_n)
    c.max_items, c.image, c.tile_last = mx, image_ptr, L.ptr(st.ch_last)
    c.unroll2 = 1 if unroll2(n_tiles) else 0
    return c


def chunk_items(st, n_tiles: int) -> None:
    """The backward's work items from the forward's per-quadrant last
    positions (isg_chunk_items), in the heaviest-first tile order."""
    if st.chunks is None or st.chunks.chunk == 0:
        return
    split = 1 if n_tiles <= SPLIT_TILES else 0
    L.check(L.lib().isg_chunk_items(n_tiles, L.ptr(st.offsets), L.ptr(st.tile_order),
                                    L.ptr(st.ch_last), st.chunks.chunk, split,
                                    L.ptr(st.ch_items), L.ptr(st.ch_n), L.stream_ptr()),
            "isg_chunk_items")


def update_params(cloud: GaussianCloud, m: dict, v: dict, grads: dict, seen, grad_accum, flag,
                  grad2d, cam_struct, lrs: list, it: int, width: int, height: int,
                  timer=None, rank_of=None, fold=None, keep_grads: bool = False) -> None:
    """Chain rule + TrainStats (isg_chain_train), then dense Adam over the five
    groups in one launch (isg_adam_groups): engine.py:508-536, optim.py:20-56.
    fold: the Rasterizer whose live subtotals the chain folds itself
    (isg_chain_fold_train; grad2d then only receives the 2-D gradients when
    fold.keep_grad2d).  FUSE_ADAM: the chain and Adam in one pass
    (isg_chain_fold_adam / isg_chain_adam_train); the parameter gradients are
    then only stored when asked for (fold.keep_grads / keep_grad2d, keep_grads)."""
    lib = L.lib()
    s = L.stream_ptr()
    p = L.Params_t()
    p.positions, p.log_scales = L.ptr(cloud.positions), L.ptr(cloud.log_scales)
    p.rotations, p.opacity_logits = L.ptr(cloud.rotations), L.ptr(cloud.opacity_logits)
    p.sh, p.n, p.degree, p.dtype = L.ptr(cloud.sh_coeffs), cloud.count, cloud.degree, L.ISG_F32
    if cloud.count == 0:
        return
    if FUSE_ADAM and (fold is not None or rank_of is None):
        # one pass: (fold +) chain + stats + Adam, gradients kept in registers
        st = L.TrainState_t()
        for k, f in zip(PARAM_NAMES, ("positions", "log_scales", "rotations", "opacity_logits",
                                      "sh")):
            setattr(st, f, L.ptr(getattr(cloud, k)))
            setattr(st, "m_" + f, L.ptr(m[k]))
            setattr(st, "v_" + f, L.ptr(v[k]))
        st.seen, st.grad_accum = L.ptr(seen), L.ptr(grad_accum)
        st.n, st.degree = cloud.count, cloud.degree
        keep = fold.keep_grad2d or fold.keep_grads if fold is not None else keep_grads
        go = (ctypes.c_void_p * 5)(*(L.ptr(grads[k]) for k in PARAM_NAMES)) if keep else None
        ll = (ctypes.c_float * 5)(*(float(np.float32(x)) for x in lrs))
        c = adam_consts(torch.float32, it, 0.0)
        if fold is not None:
            L.check(lib.isg_chain_fold_adam(
                ctypes.byref(st), ctypes.byref(cam_struct), L.ptr(rank_of), L.ptr(fold.live_off),
                L.ptr(fold.partials), L.ptr(fold.rect_sorted), 0, fold.tiles_y, fold.canon_rows,
                L.ptr(grad2d) if fold.keep_grad2d else None, go, ll, ctypes.byref(c),
                0.5 * width, 0.5 * height, s), "isg_chain_fold_adam")
        else:
            L.check(lib.isg_chain_adam_train(
                ctypes.byref(st), ctypes.byref(cam_struct), L.ptr(flag), L.ptr(grad2d), go, ll,
                ctypes.byref(c), 0.5 * width, 0.5 * height, s), "isg_chain_adam_train")
        _mark(timer, "chain")
        _mark(timer, "adam")
        return
    if fold is not None:
        L.check(lib.isg_chain_fold_train(
            ctypes.byref(p), ctypes.byref(cam_struct), L.ptr(rank_of), L.ptr(fold.live_off),
            L.ptr(fold.partials), L.ptr(fold.rect_sorted), 0, fold.tiles_y, fold.canon_rows,
            L.ptr(grad2d) if fold.keep_grad2d else None,
            L.ptr(grads["positions"]), L.ptr(grads["log_scales"]), L.ptr(grads["rotations"]),
            L.ptr(grads["opacity_logits"]), L.ptr(grads["sh_coeffs"]), L.ptr(seen),
            L.ptr(grad_accum), 0.5 * width, 0.5 * height, s), "isg_chain_fold_train")
    elif rank_of is not None:
        L.check(lib.isg_chain_train_ranked(
            ctypes.byref(p), ctypes.byref(cam_struct), L.ptr(rank_of), L.ptr(grad2d),
            L.ptr(grads["positions"]), L.ptr(grads["log_scales"]), L.ptr(grads["rotations"]),
            L.ptr(grads["opacity_logits"]), L.ptr(grads["sh_coeffs"]), L.ptr(seen),
            L.ptr(grad_accum), 0.5 * width, 0.5 * height, s), "isg_chain_train_ranked")
    else:
        L.check(lib.isg_chain_train(ctypes.byref(p), ctypes.byref(cam_struct), L.ptr(flag),
                                    L.ptr(grad2d), L.ptr(grads["positions"]),
                                    L.ptr(grads["log_scales"]), L.ptr(grads["rotations"]),
                                    L.ptr(grads["opacity_logits"]), L.ptr(grads["sh_coeffs"]),
                                    L.ptr(seen), L.ptr(grad_accum), 0.5 * width, 0.5 * height,
                                    s), "isg_chain_train")
    _mark(timer, "chain")
    P5 = ctypes.c_void_p * 5
    pp = P5(*(L.ptr(getattr(cloud, k)) for k in PARAM_NAMES))
    gg = P5(*(L.ptr(grads[k]) for k in PARAM_NAMES))
    mm = P5(*(L.ptr(m[k]) for k in PARAM_NAMES))
    vv = P5(*(L.ptr(v[k]) for k in PARAM_NAMES))
    nn = (ctypes.c_int64 * 5)(*(getattr(cloud, k).numel() for k in PARAM_NAMES))
    ll = (ctypes.c_float * 5)(*(float(np.float32(x)) for x in lrs))
    c = adam_consts(torch.float32, it, 0.0)
    L.check(lib.isg_adam_groups(5, pp, gg, mm, vv, nn, ll, ctypes.byref(c), s),
            "isg_adam_groups")
    _mark(timer, "adam")


class Trainer:
    """Single-GPU training state: parameters, Adam moments, stats, buffers."""

    def __init__(self, cloud: GaussianCloud, width: int, height: int, config: TrainConfig,
                 scene_extent: float, device=None, canon_rows: int = CANON_ROWS):
        self.device = device or L.require_cuda()
        self.cfg = config
        self.cloud = cloud
        self.scene_extent = float(scene_extent)
        n = cloud.count
        self.m = {k: torch.zeros_like(getattr(cloud, k)) for k in PARAM_NAMES}
        self.v = {k: torch.zeros_like(getattr(cloud, k)) for k in PARAM_NAMES}
        self.stats = TrainStats(grad_accum=torch.zeros(n, dtype=torch.float64, device=self.device),
                                seen=torch.zeros(n, dtype=torch.int64, device=self.device))
        self.r = Rasterizer(n, width, height, self.device, config.background,
                            canon_rows=canon_rows)
        self.r.ranked_grads = True
        self.loss_dev = torch.zeros(max(config.iterations, 1) + 1, dtype=torch.float64,
                                    device=self.device)
        self.lr_host = (ctypes.c_float * 5)()
        self.grads = None

    def _state_struct(self) -> L.TrainState_t:
        st = L.TrainState_t()
        c = self.cloud
        st.positions, st.log_scales, st.rotations = L.ptr(c.positions), L.ptr(c.log_scales), L.ptr(c.rotations)
        st.opacity_logits, st.sh = L.ptr(c.opacity_logits), L.ptr(c.sh_coeffs)
        for pre, d in (("m_", self.m), ("v_", self.v)):
            setattr(st, pre + "positions", L.ptr(d["positions"]))
            setattr(st, pre + "log_scales", L.ptr(d["log_scales"]))
            setattr(st, pre + "rotations", L.ptr(d["rotations"]))
            setattr(st, pre + "opacity_logits", L.ptr(d["opacity_logits"]))
            setattr(st, pre + "sh", L.ptr(d["sh_coeffs"]))
        st.seen, st.grad_accum = L.ptr(self.stats.seen), L.ptr(self.stats.grad_accum)
        st.n, st.degree = c.count, c.degree
        return st

    def lrs(self, it: int) -> list[float]:
        """engine.py:525-535."""
        cfg = self.cfg
        return [self.scene_extent * position_lr(cfg.lr_position, it, cfg.iterations,
                                                cfg.lr_position_final),
                cfg.lr_scale, cfg.lr_rotation, cfg.lr_opacity, cfg.lr_sh]

    def step(self, it: int, cam, gt: torch.Tensor, loss_slot: torch.Tensor | None = None) -> None:
        """One training iteration on view `cam` with ground truth `gt`
        (H, W, 3) float32 on the device.  The loss lands in loss_slot (or
        self.loss_dev[it])."""
        if it < 1:
            raise ValueError(f"iteration must be >= 1, got {it}")  # optim.py:36-38
        if loss_slot is None and it >= self.loss_dev.numel():
            # resumed / extended runs: grow the per-iteration loss record
            grown = torch.zeros(it + 1, dtype=torch.float64, device=self.device)
            grown[:self.loss_dev.numel()] = self.loss_dev
            self.loss_dev = grown
        r = self.r
        ctx = r.forward(self.cloud, cam)
        slot = loss_slot if loss_slot is not None else self.loss_dev[it:it + 1]
        loss_l1_dssim_device(r.image, gt, self.cfg.lambda_dssim, r.dl, slot)
        _mark(r.timer, "loss")
        r.backward(ctx)
        if self.grads is None:
            self.grads = {k: torch.empty_like(getattr(self.cloud, k)) for k in PARAM_NAMES}
        fused = r.live and r.fuse_fold and r.ranked_grads
        update_params(self.cloud, self.m, self.v, self.grads, self.stats.seen,
                      self.stats.grad_accum, r.flag, r.grad2d, r.cam_struct, self.lrs(it), it,
                      r.width, r.height, r.timer, rank_of=r.rank_of,
                      fold=r if fused else None)

    def densify_due(self, it: int) -> bool:
        """engine.py:540-541."""
        cfg = self.cfg
        return (cfg.densify and cfg.densify_start <= it <= cfg.effective_densify_stop()
                and it % cfg.densify_interval == 0)

    def densify(self, it: int) -> None:
        """Single-worker _densify_step (engine.py:307-382): densify_and_prune
        with global ids = row indices, Adam moments of kept rows carried, new
        rows cold, statistics restarted (a fresh _Shard)."""
        from .densify import SPLIT_EXTENT_FRACTION, carry_moments, densify_and_prune
        cfg = self.cfg
        res = cfg.resolution if cfg.resolution is not None else self.r.width
        grad_thr = cfg.effective_grad_threshold(res)
        split_thr = (cfg.split_threshold if cfg.split_threshold is not None
                     else SPLIT_EXTENT_FRACTION * self.scene_extent)
        new, mapping = densify_and_prune(self.cloud, self.stats, cfg, it, grad_thr, split_thr)
        self.m = carry_moments(self.m, mapping, new)
        self.v = carry_moments(self.v, mapping, new)
        self.cloud = new
        n = new.count
        self.stats = TrainStats(grad_accum=torch.zeros(n, dtype=torch.float64, device=self.device),
                                seen=torch.zeros(n, dtype=torch.int64, device=self.device))
        self.grads = None

    def render(self, cam) -> torch.Tensor:
        self.r.forward(self.cloud, cam)
        return self.r.image

    def evaluate(self, cameras, images_dev, it: int, wall_s: float) -> EvalRecord:
        """engine.py:440-462 + training.py:392-396 (8-bit round trip)."""
        losses, psnrs, ssims = [], [], []
        tmp_loss = torch.zeros(1, dtype=torch.float64, device=self.device)
        for v, cam in enumerate(cameras):
            img = self.render(cam)
            ref = images_dev[v]
            loss_l1_dssim_device(img, ref, self.cfg.lambda_dssim, self.r.dl, tmp_loss)
            losses.append(float(tmp_loss.item()))
            a = quantize8(img)
            b = quantize8(ref)
            psnrs.append(psnr(a, b))
            ssims.append(ssim(a, b))
        return EvalRecord(iteration=it, loss=float(np.mean(losses)), psnr=float(np.mean(psnrs)),
                          ssim=float(np.mean(ssims)), wall_s=wall_s, gaussians=self.cloud.count)


def _images_to_device(images, device) -> torch.Tensor:
    arr = images if isinstance(images, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(images))
    if arr.dtype == torch.uint8:
        arr = (arr.to(torch.float64) / 255.0).to(torch.float32)
    return arr.to(device=device, dtype=torch.float32).contiguous()


def run_training(dataset: TrainDataset, config: TrainConfig, workers: int = 1,
                 init_cloud=None, evaluate: bool = True):
    """Train a Gaussian cloud against the dataset views (engine.py:613-652).

    workers > 1 runs the sharded multi-GPU engine (distributed.py) under
    torch.distributed; workers == 1 is the single-GPU loop here.
    Returns (GaussianCloud on the device, TrainReport)."""
    config.validate()
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if config.resolution is not None and config.resolution != dataset.width:
        raise ValueError(f"config resolution {config.resolution} != dataset width {dataset.width}")
    if workers > 1:
        from .distributed import run_training_distributed
        return run_training_distributed(dataset, config, workers, init_cloud, evaluate)
    dev = L.require_cuda()
    if init_cloud is None:
        pts = np.asarray(dataset.points.positions, dtype=np.float64)
        cloud = cloud_from_points(pts, init_log_scales(pts), config.sh_degree, dev)
    else:
        cloud = to_device_cloud(init_cloud, dev, torch.float32)
    tr = Trainer(cloud, dataset.width, dataset.height, config, dataset.scene_extent, dev)
    images = _images_to_device(dataset.images, dev)
    report = TrainReport(workers=1, resolution=config.resolution or dataset.width)
    if evaluate:
        report.records.append(tr.evaluate(dataset.cameras, images, 0, 0.0))
    schedule = build_schedule(config.iterations, dataset.view_count, config.seed)
    wall = 0.0
    for it in range(1, config.iterations + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        v = schedule[it - 1]
        tr.step(it, dataset.cameras[v], images[v])
        if tr.densify_due(it):
            tr.densify(it)
        torch.cuda.synchronize()
        wall += time.perf_counter() - t0
        due = it == config.iterations or (config.eval_interval > 0 and it % config.eval_interval == 0)
        if evaluate and due:
            report.records.append(tr.evaluate(dataset.cameras, images, it, wall))
    report.iteration_losses = [float(x) for x in tr.loss_dev[1:config.iterations + 1].tolist()]
    report.total_wall_s = wall
    return tr.cloud, report


def train_single(dataset: TrainDataset, config: TrainConfig, **kw):
    """Single-GPU training (training.py:399-402)."""
    return run_training(dataset, config, workers=1, **kw)
