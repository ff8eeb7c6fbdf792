"""Sharded multi-GPU training step (reference distributed.py + engine.py W>1).

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  Each GPU
owns a contiguous shard of Gaussians (partition_gaussians, distributed.py:
72-88) and a contiguous ROW BAND of image tiles (partition_pixels; the
reference's round-robin tiles ship 2.3x more splat records at 8 GPUs, SURVEY
§8e).  One iteration, per rank, is a fixed sequence of phases separated by
collectives -- the reference's barrier-separated phases (engine.py:184-537):

  project   isg_preprocess on the shard, isg_route_* -> 80 B splat records
            grouped by destination band                      -> all-to-all #1
  render    unpack, depth sort, bin the band's tiles, raster forward into a
            window buffer                                    -> halo rows
  loss      isg_loss_rows on the band (+16/+10 halo rows); block partials of
            the loss                                         -> all-reduce
  backward  raster backward on the band, per-(splat, canonical block) fold,
            records grouped by owner shard                   -> all-to-all #2
  update    owner fold (bands ascending), chain rule + stats + Adam on the
            shard (isg_chain_adam)

Every cross-GPU meeting point has a canonical order (global (depth, id) sort;
canonical 8-tile-row blocks summed in band order; fixed-order loss sums), so
the result is bitwise identical for any GPU count (tests/test_dist_gpu.py
checks W = 1, 2, 3 against the single-GPU engine on one B200 by running the
ranks' phases in sequence with an in-process exchange).

The reference's public data-plane API (ShardMap, partition_gaussians,
PixelPartition, partition_pixels, route_rows, GradChunk/GradMessage,
reduce_gradients_fused, ProtocolError, estimate_min_workers) is kept here with
the same names and error behaviour.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L

TILE = 16
CANON_ROWS = 8
# our kernels per sharded step (CUB scan/sort passes not counted): preprocess,
# route_count, route_emit, dest offsets, route_gather | records_unpack,
# depth tie fix, gather_rank, finish_counts, bin_emit16_cull, tile_offsets16,
# raster_fwd_masked | ssim_fields, ssim_adjoint, loss_finish | raster_bwd_masked,
# block_count, block_fold, owner offsets, grad_gather | grad_rows, seg
# offsets, owner_fold, chain_train, adam_groups
LAUNCHES_PER_STEP = 24


class ProtocolError(RuntimeError):
    """A message violated the exchange contract (bad owner, duplicate tile)."""


# ------------------------------------------------------ reference data plane --

@dataclass
class ShardMap:
    """Assignment of Gaussian rows to workers (distributed.py:23-69)."""

    workers: int
    owner: np.ndarray
    lists: list

    @classmethod
    def from_lists(cls, lists, n: int) -> "ShardMap":
        owner = np.full(n, -1, dtype=np.int32)
        for w, ids in enumerate(lists):
            owner[np.asarray(ids, dtype=np.int64)] = w
        m = cls(workers=len(lists), owner=owner,
                lists=[np.asarray(l, dtype=np.int64) for l in lists])
        m.validate()
        return m

    @property
    def total(self) -> int:
        return int(self.owner.shape[0])

    @property
    def sizes(self) -> list:
        return [int(l.shape[0]) for l in self.lists]

    @property
    def starts(self) -> list:
        """Contiguous-shard boundaries (n_workers + 1)."""
        out = [0]
        for s in self.sizes:
            out.append(out[-1] + s)
        return out

    def validate(self) -> None:
        n = self.total
        if self.workers < 1 or len(self.lists) != self.workers:
            raise ValueError("worker count does not match shard lists")
        seen = np.zeros(n, dtype=bool)
        for w, ids in enumerate(self.lists):
            if ids.size and (np.diff(ids) <= 0).any():
                raise ValueError(f"shard {w} ids not strictly ascending")
            if ids.size and (ids[0] < 0 or ids[-1] >= n):
                raise ValueError(f"shard {w} ids out of range")
            if seen[ids].any():
                raise ValueError("shard lists overlap")
            seen[ids] = True
            if not (self.owner[ids] == w).all():
                raise ValueError("owner array disagrees with shard lists")
        if not seen.all():
            raise ValueError("shard lists do not cover every row")


def partition_gaussians(n: int, workers: int, strategy: str = "contiguous-balanced") -> ShardMap:
    """Contiguous shards with sizes differing by at most one (distributed.py:72-88)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if n < 0:
        raise ValueError("n must be >= 0")
    if strategy != "contiguous-balanced":
        raise ValueError(f"unknown strategy {strategy!r}")
    base, rem = divmod(n, workers)
    lists, start = [], 0
    for w in range(workers):
        size = base + (1 if w < rem else 0)
        lists.append(np.arange(start, start + size, dtype=np.int64))
        start += size
    return ShardMap.from_lists(lists, n)


@dataclass
class PixelPartition:
    """Row-band assignment of image tiles to workers.

    band_rows[w]..band_rows[w+1] are worker w's tile rows; each band is a union
    of whole canonical blocks of `canon_rows` tile rows (the W-independent fold
    grouping).  `assignment` (tile id -> worker) mirrors the reference's
    PixelPartition (distributed.py:91-108)."""

    width: int
    height: int
    tile_size: int
    workers: int
    tiles_x: int
    tiles_y: int
    band_rows: list
    canon_rows: int = CANON_ROWS

    @property
    def tile_count(self) -> int:
        return self.tiles_x * self.tiles_y

    @property
    def assignment(self) -> np.ndarray:
        a = np.empty(self.tile_count, dtype=np.int32)
        for w in range(self.workers):
            a[self.band_rows[w] * self.tiles_x:self.band_rows[w + 1] * self.tiles_x] = w
        return a

    def tiles_of(self, worker: int) -> np.ndarray:
        return np.arange(self.band_rows[worker] * self.tiles_x,
                         self.band_rows[worker + 1] * self.tiles_x, dtype=np.int32)

    def pixel_rows(self, worker: int) -> tuple:
        return (self.band_rows[worker] * self.tile_size,
                min(self.band_rows[worker + 1] * self.tile_size, self.height))


def partition_pixels(width: int, height: int, tile_size: int, workers: int,
                     canon_rows: int = CANON_ROWS, weights=None) -> PixelPartition:
    """Contiguous row bands of whole canonical blocks, balanced by block count
    (or by `weights`, a per-block cost estimate)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if width < 1 or height < 1 or tile_size < 1:
        raise ValueError("image and tile dims must be positive")
    tiles_x = (width + tile_size - 1) // tile_size
    tiles_y = (height + tile_size - 1) // tile_size
    n_blocks = (tiles_y + canon_rows - 1) // canon_rows
    if n_blocks < workers:
        raise ValueError(f"{n_blocks} canonical blocks of {canon_rows} tile rows cannot feed "
                         f"{workers} workers; lower canon_rows")
    if weights is None:
        cuts = [round(w * n_blocks / workers) for w in range(workers + 1)]
    else:
        cw = np.concatenate([[0.0], np.cumsum(np.asarray(weights, dtype=np.float64))])
        cuts = [0]
        for w in range(1, workers):
            target = cw[-1] * w / workers
            b = int(np.searchsorted(cw, target))
            cuts.append(min(max(b, cuts[-1] + 1), n_blocks - (workers - w)))
        cuts.append(n_blocks)
    band_rows = [min(c * canon_rows, tiles_y) for c in cuts]
    return PixelPartition(width, height, tile_size, workers, tiles_x, tiles_y, band_rows,
                          canon_rows)


def route_rows(tile_min, tile_max, part: PixelPartition) -> np.ndarray:
    """(n, W) membership mask: row i reaches worker w iff its tile rect
    overlaps w's band (distributed.py:127-136 for row bands)."""
    tmin = np.asarray(tile_min)
    tmax = np.asarray(tile_max)
    n = tmin.shape[0]
    mask = np.zeros((n, part.workers), dtype=np.uint8)
    for w in range(part.workers):
        lo, hi = part.band_rows[w], part.band_rows[w + 1]
        mask[:, w] = ((tmin[:, 1] < hi) & (tmax[:, 1] >= lo)).astype(np.uint8)
    return mask


def estimate_min_workers(n_gaussians: int, per_worker_capacity: int) -> int:
    """distributed.py:271-277."""
    if per_worker_capacity <= 0:
        raise ValueError("per-worker capacity must be positive")
    if n_gaussians < 0:
        raise ValueError("gaussian count must be >= 0")
    return max(1, math.ceil(n_gaussians / per_worker_capacity))


@dataclass
class GradChunk:
    """One producing tile's gradient rows (distributed.py:157-166)."""

    tile_id: int
    indices: np.ndarray
    dmean2d: np.ndarray
    dconic: np.ndarray
    dcolor: np.ndarray
    dopacity: np.ndarray


@dataclass
class GradMessage:
    """distributed.py:169-175."""

    producer: int
    destination: int
    chunks: list = field(default_factory=list)


def reduce_gradients_fused(messages, shard_map: ShardMap) -> dict:
    """Sum routed gradients at each owner in ascending producing-tile order
    (distributed.py:178-226), on the device: chunks are ordered by tile id and
    folded with the owner-fold kernel (float64, arrival = tile order)."""
    per_dest: dict = {}
    pairs = set()
    for msg in messages:
        key = (msg.producer, msg.destination)
        if key in pairs:
            raise ProtocolError(f"duplicate message for pair {key}")
        pairs.add(key)
        per_dest.setdefault(msg.destination, []).extend(msg.chunks)
    out = {}
    for dest, chunks in per_dest.items():
        if not 0 <= dest < shard_map.workers:
            raise ProtocolError(f"unknown destination worker {dest}")
        owned = shard_map.lists[dest]
        n = owned.shape[0]
        seen = set()
        rows_l, vals_l = [], []
        for ch in sorted(chunks, key=lambda c: c.tile_id):
            if ch.tile_id in seen:
                raise ProtocolError(f"tile {ch.tile_id} contributed twice")
            seen.add(ch.tile_id)
            idx = np.asarray(ch.indices, dtype=np.int64)
            rows = np.searchsorted(owned, idx)
            bad = (rows >= n) | (owned[np.minimum(rows, max(n - 1, 0))] != idx) if n else \
                np.ones(idx.shape, dtype=bool)
            if bad.any():
                raise ProtocolError(f"indices {idx[bad][:4].tolist()} not owned by worker {dest}")
            rows_l.append(rows)
            vals_l.append(np.concatenate([np.asarray(ch.dmean2d).reshape(-1, 2),
                                          np.asarray(ch.dconic).reshape(-1, 3),
                                          np.asarray(ch.dcolor).reshape(-1, 3),
                                          np.asarray(ch.dopacity).reshape(-1, 1)], 1))
        dev = L.require_cuda()
        g2d = torch.zeros((n, 9), dtype=torch.float64, device=dev)
        if rows_l:
            rows = np.concatenate(rows_l).astype(np.int32)
            vals = np.concatenate(vals_l).astype(np.float64)
            rec = np.zeros((rows.shape[0], 20), dtype=np.int32)
            rec[:, 0] = rows
            rec[:, 2:] = vals.view(np.int32).reshape(-1, 18)
            g2d = _owner_fold(torch.from_numpy(rec).to(dev), n, dev, L.Workspace())
        out[dest] = {"dmean2d": g2d[:, 0:2], "dconic": g2d[:, 2:5], "dcolor": g2d[:, 5:8],
                     "dopacity": g2d[:, 8]}
    return out


def _bits(n: int) -> int:
    return max(1, int(max(n, 1) - 1).bit_length())


def _owner_fold(records: torch.Tensor, n_rows: int, dev, ws: L.Workspace,
                grad2d: torch.Tensor | None = None) -> torch.Tensor:
    """Stable group of gradient records by row, then in-order float64 sums."""
    lib = L.lib()
    s = L.stream_ptr()
    r = int(records.shape[0])
    if grad2d is None:
        grad2d = torch.zeros((n_rows, 9), dtype=torch.float64, device=dev)
    if r == 0 or n_rows == 0:
        return grad2d
    rows = torch.empty(r, dtype=torch.int32, device=dev)
    idx = torch.empty(r, dtype=torch.int32, device=dev)
    L.check(lib.isg_grad_rows(r, L.ptr(records), L.ptr(rows), L.ptr(idx), s), "isg_grad_rows")
    srows, perm = L.sort_pairs(rows, idx, (0, _bits(n_rows)), ws)
    seg = torch.empty(n_rows + 1, dtype=torch.int32, device=dev)
    L.check(lib.isg_tile_offsets(r, L.ptr(srows), n_rows, L.ptr(seg), s), "seg offsets")
    L.check(lib.isg_owner_fold(n_rows, L.ptr(seg), L.ptr(perm), L.ptr(records), L.ptr(grad2d), s),
            "isg_owner_fold")
    return grad2d


# ------------------------------------------------------------ communicators --

class TorchComm:
    """Collectives over a torch.distributed process group (NCCL on GPUs; gloo
    for the CPU tests of this layer)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def alltoallv(self, send: torch.Tensor, send_counts: list) -> tuple:
        """Rows of `send` (grouped by destination, counts per destination) ->
        received rows concatenated in source-rank order, and the counts."""
        dev = send.device
        sc = torch.tensor(send_counts, dtype=torch.int64, device=dev)
        rc = torch.empty_like(sc)
        self.dist.all_to_all_single(rc, sc, group=self.group)
        recv_counts = [int(v) for v in rc.tolist()]
        cols = send.shape[1:]
        recv = torch.empty((sum(recv_counts),) + tuple(cols), dtype=send.dtype, device=dev)
        self.dist.all_to_all_single(recv, send.contiguous(), output_split_sizes=recv_counts,
                                    input_split_sizes=list(send_counts), group=self.group)
        return recv, recv_counts

    def halo(self, to_prev: torch.Tensor | None, to_next: torch.Tensor | None,
             from_prev_shape, from_next_shape, dtype, dev) -> tuple:
        """Exchange boundary rows with the neighbouring ranks."""
        ops = []
        got_prev = got_next = None
        P2POp = self.dist.P2POp
        if self.rank > 0 and from_prev_shape is not None:
            got_prev = torch.empty(from_prev_shape, dtype=dtype, device=dev)
            ops.append(P2POp(self.dist.irecv, got_prev, self.rank - 1, self.group))
        if self.rank + 1 < self.world and from_next_shape is not None:
            got_next = torch.empty(from_next_shape, dtype=dtype, device=dev)
            ops.append(P2POp(self.dist.irecv, got_next, self.rank + 1, self.group))
        if self.rank > 0 and to_prev is not None:
            ops.append(P2POp(self.dist.isend, to_prev.contiguous(), self.rank - 1, self.group))
        if self.rank + 1 < self.world and to_next is not None:
            ops.append(P2POp(self.dist.isend, to_next.contiguous(), self.rank + 1, self.group))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        return got_prev, got_next

    def allreduce_sum_(self, t: torch.Tensor) -> torch.Tensor:
        self.dist.all_reduce(t, group=self.group)
        return t

    def max_(self, t: torch.Tensor) -> torch.Tensor:
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return t


# --------------------------------------------------------------- rank state --

class RankStep:
    """One rank's shard, band and buffers, with the phases of an iteration."""

    def __init__(self, rank: int, world: int, shards: ShardMap, part: PixelPartition,
                 params: dict, degree: int, config, scene_extent: float, device,
                 background=(1.0, 1.0, 1.0)):
        from .gaussians import GaussianCloud, PARAM_NAMES
        self.rank, self.world = rank, world
        self.dev = device
        self.cfg = config
        self.scene_extent = float(scene_extent)
        self.part = part
        self.shard_starts = shards.starts
        self.id_base = self.shard_starts[rank]
        self.cloud = GaussianCloud(*(params[k] for k in PARAM_NAMES), degree=degree)
        self.n = self.cloud.count
        self.m = {k: torch.zeros_like(params[k]) for k in PARAM_NAMES}
        self.v = {k: torch.zeros_like(params[k]) for k in PARAM_NAMES}
        self.seen = torch.zeros(self.n, dtype=torch.int64, device=device)
        self.grad_accum = torch.zeros(self.n, dtype=torch.float64, device=device)
        self.W, self.H = part.width, part.height
        self.tiles_x = part.tiles_x
        self.trow0, self.trow1 = part.band_rows[rank], part.band_rows[rank + 1]
        self.prow0, self.prow1 = part.pixel_rows(rank)
        self.win0 = max(0, self.prow0 - 16)
        self.win1 = min(self.H, self.prow1 + 10)
        self.bg = (ctypes.c_double * 3)(*[float(v) for v in background])
        self.band_host = (ctypes.c_int32 * (world + 1))(*part.band_rows)
        self.shard_host = (ctypes.c_int64 * (world + 1))(*self.shard_starts)
        n_tiles = (self.trow1 - self.trow0) * self.tiles_x
        self.n_tiles = n_tiles
        self.tile_bits = _bits(n_tiles)
        d = device
        n = self.n
        # shard-side buffers
        self.key = torch.empty(n, dtype=torch.int64, device=d)
        self.rect = torch.empty((n, 4), dtype=torch.int32, device=d)
        self.feat = torch.empty((n, 12), dtype=torch.float32, device=d)
        self.flag = torch.empty(n, dtype=torch.uint8, device=d)
        self.cnt = torch.empty(n, dtype=torch.int64, device=d)
        self.dlo = torch.empty(n, dtype=torch.int32, device=d)
        self.roff = torch.empty(n + 1, dtype=torch.int64, device=d)
        self.grad2d = torch.zeros((n, 9), dtype=torch.float64, device=d)
        self.total = torch.zeros(1, dtype=torch.int64, device=d)
        self.counts = torch.zeros(2, dtype=torch.int64, device=d)
        self.host = torch.zeros(4, dtype=torch.int64).pin_memory()
        rows = self.win1 - self.win0
        self.window = torch.zeros((max(rows, 1), self.W, 3), dtype=torch.float32, device=d)
        band_px = (self.prow1 - self.prow0) * self.W
        self.t_final = torch.empty(max(band_px, 1), dtype=torch.float32, device=d)
        self.n_last = torch.empty(max(band_px, 1), dtype=torch.int32, device=d)
        self.dl = torch.empty((max(band_px, 1), 3), dtype=torch.float32, device=d)
        self.offsets = torch.empty(n_tiles + 1, dtype=torch.int32, device=d)
        nf = ctypes.c_int32(0)
        na = ctypes.c_int32(0)
        L.lib().isg_loss_partials_size(self.H, self.W, ctypes.byref(nf), ctypes.byref(na))
        self.n_ps, self.n_pl = nf.value, na.value
        self.parts = torch.zeros(self.n_ps + self.n_pl, dtype=torch.float64, device=d)
        self.loss_dev = torch.zeros(1, dtype=torch.float64, device=d)
        self.ws = [L.Workspace() for _ in range(4)]
        self.lr_host = (ctypes.c_float * 5)()

    # -- helpers --------------------------------------------------------
    def _sync_ints(self, *tensors) -> list:
        k = 0
        for t in tensors:
            self.host[k:k + t.numel()].copy_(t, non_blocking=True)
            k += t.numel()
        torch.cuda.current_stream().synchronize()
        return [int(v) for v in self.host[:k].tolist()]

    def _vptr(self, t: torch.Tensor, row0: int, row_elems: int) -> int:
        """Virtual base pointer so that global row `row0` maps to t's start."""
        return t.data_ptr() - row0 * row_elems * t.element_size()

    # -- phase 1: project + route ----------------------------------------
    def phase_project(self, cam):
        lib, s, d = L.lib(), L.stream_ptr(), self.dev
        c = self.cloud
        self.cam_struct = L.camera_struct(cam)
        if self.n:
            p = L.Params_t()
            p.positions, p.log_scales = L.ptr(c.positions), L.ptr(c.log_scales)
            p.rotations, p.opacity_logits = L.ptr(c.rotations), L.ptr(c.opacity_logits)
            p.sh, p.n, p.degree, p.dtype = L.ptr(c.sh_coeffs), self.n, c.degree, L.ISG_F32
            out = L.PreprocessOut_t()
            out.key, out.rect, out.feat = L.ptr(self.key), L.ptr(self.rect), L.ptr(self.feat)
            out.flag, out.full64, out.feat_dtype = L.ptr(self.flag), None, L.ISG_F32
            L.check(lib.isg_preprocess(ctypes.byref(p), ctypes.byref(self.cam_struct), TILE,
                                       ctypes.byref(out), s), "isg_preprocess")
            L.check(lib.isg_route_count(self.n, L.ptr(self.flag), L.ptr(self.rect),
                                        self.band_host, self.world, L.ptr(self.cnt),
                                        L.ptr(self.dlo), s), "isg_route_count")
        self._scan(self.n, self.cnt, self.roff, self.total)
        (S,) = self._sync_ints(self.total)
        keys = torch.empty(max(S, 1), dtype=torch.int32, device=d)
        vals = torch.empty(max(S, 1), dtype=torch.int32, device=d)
        if S:
            L.check(lib.isg_route_emit(self.n, L.ptr(self.roff), L.ptr(self.dlo), L.ptr(keys),
                                       L.ptr(vals), s), "isg_route_emit")
            keys, vals = L.sort_pairs(keys[:S], vals[:S], (0, _bits(self.world)), self.ws[0])
        doff = torch.empty(self.world + 1, dtype=torch.int32, device=d)
        L.check(lib.isg_tile_offsets(S, L.ptr(keys), self.world, L.ptr(doff), s), "dest offsets")
        rec = torch.empty((max(S, 1), 20), dtype=torch.int32, device=d)
        if S:
            L.check(lib.isg_route_gather(S, L.ptr(vals), L.ptr(self.key), L.ptr(self.rect),
                                         L.ptr(self.feat), self.id_base, L.ptr(rec), s),
                    "isg_route_gather")
        counts = (doff[1:] - doff[:-1]).tolist()
        return rec[:S], [int(v) for v in counts]

    def _scan(self, n, cnt, off, total):
        lib = L.lib()
        sz = ctypes.c_size_t(0)
        L.check(lib.isg_scan_i64(None, ctypes.byref(sz), n, None, None, None, None), "scan size")
        buf = self.ws[1].get(sz.value, self.dev)
        sz = ctypes.c_size_t(buf.numel())
        L.check(lib.isg_scan_i64(L.ptr(buf), ctypes.byref(sz), n, L.ptr(cnt), L.ptr(off),
                                 L.ptr(total), L.stream_ptr()), "isg_scan_i64")

    # -- phase 2: render the band -----------------------------------------
    def phase_render(self, records: torch.Tensor, count: bool = False):
        """count=True: the reference's full band lists and the unmasked
        forward with per-pixel pair counters (n_contrib, n_iter; n_last is
        then the full-list last-contributor index) for the roofline units;
        leaves no state for a backward."""
        lib, s, d = L.lib(), L.stream_ptr(), self.dev
        R = int(records.shape[0])
        self.R = R
        self.r_key = torch.empty(max(R, 1), dtype=torch.int64, device=d)
        self.r_gid = torch.empty(max(R, 1), dtype=torch.int32, device=d)
        self.r_rect = torch.empty((max(R, 1), 4), dtype=torch.int32, device=d)
        self.r_feat = torch.empty((max(R, 1), 12), dtype=torch.float32, device=d)
        L.check(lib.isg_records_unpack(R, L.ptr(records), L.ptr(self.r_key), L.ptr(self.r_gid),
                                       L.ptr(self.r_rect), L.ptr(self.r_feat), s), "unpack")
        vals0 = torch.arange(max(R, 1), dtype=torch.int32, device=d)
        self.key_sorted, self.order = L.sort_depth(self.r_key[:R], vals0[:R], self.ws[0])
        self.rect_sorted = torch.empty((max(R, 1), 4), dtype=torch.int32, device=d)
        self.feat_sorted = torch.empty((max(R, 1), 12), dtype=torch.float32, device=d)
        self.emit_off = torch.empty(R + 1, dtype=torch.int64, device=d)
        sz = ctypes.c_size_t(0)
        L.check(lib.isg_bin_count(None, ctypes.byref(sz), R, None, None, None, None, L.ISG_F32,
                                  self.trow0, self.trow1, None, None, None, None, None), "bin size")
        ws = self.ws[2].get(sz.value, d)
        sz = ctypes.c_size_t(ws.numel())
        L.check(lib.isg_bin_count(L.ptr(ws), ctypes.byref(sz), R, L.ptr(self.key_sorted),
                                  L.ptr(self.order), L.ptr(self.r_rect), L.ptr(self.r_feat),
                                  L.ISG_F32, self.trow0, self.trow1, L.ptr(self.rect_sorted),
                                  L.ptr(self.feat_sorted), L.ptr(self.emit_off),
                                  L.ptr(self.counts), s), "isg_bin_count")
        M, E = self._sync_ints(self.counts)
        self.M, self.E = M, E
        k16 = self.n_tiles <= 65536  # 2-byte tile keys (see engine.Rasterizer.forward)
        tk = torch.empty(max(E, 1), dtype=torch.int16 if k16 else torch.int32, device=d)
        tv = torch.empty(max(E, 1), dtype=torch.int32, device=d)
        emit = lib.isg_bin_emit16 if k16 else lib.isg_bin_emit
        offs = lib.isg_tile_offsets16 if k16 else lib.isg_tile_offsets
        # band lists leave out the pairs no pixel of their tile can composite
        # (isg_bin_emit16_cull writes their zero subtotals; see engine.Rasterizer)
        cull = self.n_tiles < 65536 and not count
        self.partials = torch.empty((max(E, 1), 12), dtype=torch.float32, device=d)
        if E:
            if cull:
                L.check(lib.isg_bin_emit16_cull(M, L.ptr(self.rect_sorted), L.ptr(self.emit_off),
                                                L.ptr(self.feat_sorted), self.tiles_x, self.trow0,
                                                self.trow1, L.ptr(tk), L.ptr(tv),
                                                L.ptr(self.partials), s), "isg_bin_emit16_cull")
            else:
                L.check(emit(M, L.ptr(self.rect_sorted), L.ptr(self.emit_off), self.tiles_x,
                             self.trow0, self.trow1, L.ptr(tk), L.ptr(tv), s), "isg_bin_emit")
            bits = max(self.tile_bits, int(self.n_tiles).bit_length()) if cull else self.tile_bits
            tk, tv = L.sort_pairs(tk[:E], tv[:E], (0, bits), self.ws[0])
        self.entries = tv
        L.check(offs(E, L.ptr(tk), self.n_tiles, L.ptr(self.offsets), s), "isg_tile_offsets")
        W3 = self.W * 3
        if count:
            band_px = max((self.prow1 - self.prow0) * self.W, 1)
            self.n_contrib = torch.zeros(band_px, dtype=torch.int32, device=d)
            self.n_iter = torch.zeros(band_px, dtype=torch.int32, device=d)
            if self.n_tiles:
                L.check(lib.isg_raster_fwd(
                    L.ISG_F32, self.W, self.H, self.tiles_x, self.trow0, self.trow1, None, 0,
                    L.ptr(self.offsets), L.ptr(self.entries), L.ptr(self.feat_sorted),
                    ctypes.cast(self.bg, ctypes.c_void_p),
                    self._vptr(self.window, self.win0, W3), L.ISG_F32,
                    self._vptr(self.t_final, self.prow0, self.W),
                    self._vptr(self.n_last, self.prow0, self.W),
                    self._vptr(self.n_contrib, self.prow0, self.W),
                    self._vptr(self.n_iter, self.prow0, self.W), None, s), "isg_raster_fwd")
            return None, None
        if self.n_tiles:
            # contribution masks for the band's backward (isg_raster_bwd_masked)
            self.cmask = torch.empty(lib.isg_contrib_mask_words(E, self.n_tiles),
                                     dtype=torch.int32, device=d)
            L.check(lib.isg_raster_fwd_masked(
                self.W, self.H, self.tiles_x, self.trow0, self.trow1, None, 0,
                L.ptr(self.offsets), L.ptr(self.entries), L.ptr(self.feat_sorted),
                ctypes.cast(self.bg, ctypes.c_void_p),
                self._vptr(self.window, self.win0, W3), L.ISG_F32,
                self._vptr(self.t_final, self.prow0, self.W),
                self._vptr(self.n_last, self.prow0, self.W), None, None, None, L.ptr(self.cmask),
                s), "isg_raster_fwd_masked")
        # boundary rows for the neighbours' SSIM halo
        b0, b1 = self.prow0 - self.win0, self.prow1 - self.win0
        to_prev = self.window[b0:b0 + min(10, b1 - b0)] if self.rank > 0 else None
        to_next = self.window[max(b0, b1 - 16):b1] if self.rank + 1 < self.world else None
        return to_prev, to_next

    def halo_shapes(self):
        prev = (self.prow0 - self.win0, self.W, 3) if self.rank > 0 else None
        nxt = (self.win1 - self.prow1, self.W, 3) if self.rank + 1 < self.world else None
        return prev, nxt

    # -- phase 3: loss on the band ----------------------------------------
    def phase_loss(self, from_prev, from_next, gt: torch.Tensor):
        lib, s = L.lib(), L.stream_ptr()
        if from_prev is not None and from_prev.shape[0]:
            self.window[:from_prev.shape[0]].copy_(from_prev)
        if from_next is not None and from_next.shape[0]:
            self.window[self.prow1 - self.win0:].copy_(from_next)
        self.parts.zero_()
        u8 = 1 if gt.dtype == torch.uint8 else 0
        if self.prow1 > self.prow0:
            sz = ctypes.c_size_t(0)
            L.check(lib.isg_loss_rows(None, ctypes.byref(sz), L.ISG_F32, self.H, self.W,
                                      self.prow0, self.prow1, None, 0, None, u8,
                                      float(self.cfg.lambda_dssim), None, None, None, None),
                    "loss size")
            buf = self.ws[3].get(sz.value, self.dev)
            sz = ctypes.c_size_t(buf.numel())
            L.check(lib.isg_loss_rows(L.ptr(buf), ctypes.byref(sz), L.ISG_F32, self.H, self.W,
                                      self.prow0, self.prow1, L.ptr(self.window), self.win0,
                                      L.ptr(gt), u8, float(self.cfg.lambda_dssim),
                                      L.ptr(self.dl), L.ptr(self.parts),
                                      self.parts.data_ptr() + 8 * self.n_ps, s), "isg_loss_rows")
        return self.parts

    def finish_loss(self):
        L.check(L.lib().isg_loss_finish(self.H, self.W, float(self.cfg.lambda_dssim),
                                        L.ptr(self.parts), self.parts.data_ptr() + 8 * self.n_ps,
                                        L.ptr(self.loss_dev), L.stream_ptr()), "isg_loss_finish")
        return self.loss_dev

    # -- phase 4: backward + per-block records for the owners --------------
    def phase_backward(self, timer=None):
        from .engine import _mark
        lib, s, d = L.lib(), L.stream_ptr(), self.dev
        E, M = self.E, self.M
        W3 = self.W * 3
        if self.n_tiles:
            L.check(lib.isg_raster_bwd_masked(
                self.W, self.H, self.tiles_x, self.trow0, self.trow1, None, 0,
                L.ptr(self.offsets), L.ptr(self.entries), L.ptr(self.feat_sorted),
                L.ptr(self.rect_sorted), L.ptr(self.emit_off), ctypes.cast(self.bg, ctypes.c_void_p),
                self._vptr(self.t_final, self.prow0, self.W),
                self._vptr(self.n_last, self.prow0, self.W),
                self._vptr(self.dl, self.prow0, W3), L.ISG_F32, L.ptr(self.partials),
                L.ptr(self.cmask), s), "isg_raster_bwd_masked")
        _mark(timer, "raster_bwd")
        nb = torch.empty(max(M, 1), dtype=torch.int64, device=d)
        rec_off = torch.empty(M + 1, dtype=torch.int64, device=d)
        if M:
            L.check(lib.isg_block_count(M, L.ptr(self.rect_sorted), self.trow0, self.trow1,
                                        self.part.canon_rows, L.ptr(nb), s), "isg_block_count")
        self._scan(M, nb, rec_off, self.total)
        (NR,) = self._sync_ints(self.total)
        owner = torch.empty(max(NR, 1), dtype=torch.int32, device=d)
        rrow = torch.empty(max(NR, 1), dtype=torch.int32, device=d)
        rval = torch.empty((max(NR, 1), 9), dtype=torch.float64, device=d)
        if NR:
            L.check(lib.isg_block_fold(L.ISG_F32, M, L.ptr(self.emit_off), L.ptr(self.partials),
                                       L.ptr(self.rect_sorted), self.trow0, self.trow1,
                                       self.part.canon_rows, L.ptr(rec_off), L.ptr(self.order),
                                       L.ptr(self.r_gid), self.shard_host, self.world,
                                       L.ptr(owner), L.ptr(rrow), L.ptr(rval), s), "isg_block_fold")
        idx0 = torch.arange(max(NR, 1), dtype=torch.int32, device=d)
        okeys, oidx = owner[:NR], idx0[:NR]
        if NR:
            okeys, oidx = L.sort_pairs(owner[:NR], idx0[:NR], (0, _bits(self.world)), self.ws[0])
        doff = torch.empty(self.world + 1, dtype=torch.int32, device=d)
        L.check(lib.isg_tile_offsets(NR, L.ptr(okeys) if NR else None, self.world, L.ptr(doff), s),
                "owner offsets")
        out = torch.empty((max(NR, 1), 20), dtype=torch.int32, device=d)
        if NR:
            L.check(lib.isg_grad_gather(NR, L.ptr(oidx), L.ptr(rrow), L.ptr(rval), L.ptr(out), s),
                    "isg_grad_gather")
        counts = [int(v) for v in (doff[1:] - doff[:-1]).tolist()]
        return out[:NR], counts

    # -- phase 5: owner fold + chain + Adam -------------------------------
    def phase_update(self, grad_records: torch.Tensor, it: int):
        from .optim import adam_consts, position_lr
        _owner_fold(grad_records, self.n, self.dev, self.ws[0], self.grad2d)
        if not self.n:
            return
        cfg = self.cfg
        lrs = [self.scene_extent * position_lr(cfg.lr_position, it, cfg.iterations,
                                               cfg.lr_position_final),
               cfg.lr_scale, cfg.lr_rotation, cfg.lr_opacity, cfg.lr_sh]
        from .engine import update_params
        if getattr(self, "grads", None) is None:
            self.grads = {k: torch.empty_like(v) for k, v in self.m.items()}
        update_params(self.cloud, self.m, self.v, self.grads, self.seen, self.grad_accum,
                      self.flag, self.grad2d, self.cam_struct, lrs, it, self.W, self.H)


# ------------------------------------------------------- densify + rebalance --
# _densify_step + _rebalance_step (engine.py:307-437), for contiguous shards:
# every rank classifies its own rows (densify.classify on the rows' state,
# children seeded by (seed, iteration, global id) with global id = shard
# start + row), the per-rank class counts fix the single-worker new-id order
# (all kept rows by ascending old id, then clones by parent, then the two
# children of every split parent), the new id space is re-cut into balanced
# contiguous shards, and rows move to their new owner with one all-to-all-v.
# Kept rows carry their Adam moments; new rows start cold; the statistics of
# every rank restart at zero.  The result is bitwise the single-GPU densify.

def densify_local(rs: "RankStep", it: int, grad_threshold: float, split_threshold: float):
    """Phase 1 on one rank: classify and build this rank's outgoing rows in
    [kept, clones, children] order.  Returns (payload (R, F) float32 with the
    23 parameter floats + m + v per row, counts (n_kept, n_clone, n_split))."""
    from .densify import densify_and_prune
    from .gaussians import PARAM_NAMES
    from .training import TrainStats
    ids = np.arange(rs.id_base, rs.id_base + rs.n, dtype=np.int64)
    new, mp = densify_and_prune(rs.cloud, TrainStats(grad_accum=rs.grad_accum, seen=rs.seen),
                                rs.cfg, it, grad_threshold, split_threshold, global_ids=ids)
    nk, nc, ns = int(mp.kept.numel()), int(mp.cloned.numel()), int(mp.split.numel())
    cols = []
    for k in PARAM_NAMES:
        t = getattr(new, k)
        cols.append(t.reshape(t.shape[0], -1))
    for st in (rs.m, rs.v):
        for k in PARAM_NAMES:
            t = getattr(new, k)
            z = torch.zeros((t.shape[0], t[0].numel()), dtype=t.dtype, device=t.device)
            if nk:
                z[:nk] = st[k][mp.kept].reshape(nk, -1)
            cols.append(z)
    payload = torch.cat(cols, 1).contiguous()
    return payload, (nk, nc, ns)


def densify_targets(counts_all: list, rank: int, world: int):
    """New global ids of rank `rank`'s outgoing rows (kept, clones, children
    in order) from every rank's (kept, clone, split) counts, the new balanced
    shard map, and the number of rows this rank sends to each destination."""
    K = sum(c[0] for c in counts_all)
    C = sum(c[1] for c in counts_all)
    S = sum(c[2] for c in counts_all)
    kb = sum(c[0] for c in counts_all[:rank])
    cb = sum(c[1] for c in counts_all[:rank])
    sb = sum(c[2] for c in counts_all[:rank])
    nk, nc, ns = counts_all[rank]
    new_ids = np.concatenate([kb + np.arange(nk), K + cb + np.arange(nc),
                              K + C + 2 * sb + np.arange(2 * ns)]).astype(np.int64)
    smap = partition_gaussians(K + C + 2 * S, world)
    starts = np.asarray(smap.starts, dtype=np.int64)
    # ids ascend inside the outgoing list, so destinations are contiguous runs
    cuts = np.searchsorted(new_ids, starts, side="left")
    send_counts = [int(cuts[d + 1] - cuts[d]) for d in range(world)]
    return new_ids, smap, send_counts


def _param_width(k: str, degree: int) -> int:
    return {"positions": 3, "log_scales": 3, "rotations": 4, "opacity_logits": 1,
            "sh_coeffs": 3 * (degree + 1) ** 2}[k]


def assemble_rows(recv: torch.Tensor, recv_ids: torch.Tensor, smap: ShardMap,
                  rank: int) -> torch.Tensor:
    """The rows a rank received (any order) placed by their new global id:
    row id - shard start is the new local row; every row arrives once."""
    n_new = smap.sizes[rank]
    if recv.shape[0] != n_new:
        raise ProtocolError(f"rank {rank}: densify delivered {recv.shape[0]} rows, "
                            f"expected {n_new}")
    local = recv_ids.to(torch.int64) - smap.starts[rank]
    if n_new and (int(local.min()) < 0 or int(local.max()) >= n_new
                  or torch.unique(local).numel() != n_new):
        raise ProtocolError(f"rank {rank}: densify rows do not tile the new shard")
    rows = torch.empty_like(recv)
    rows[local] = recv
    return rows


def unpack_rows(rows: torch.Tensor, degree: int) -> list:
    """(params, m, v) dicts from the packed (R, 3 * 23) rows."""
    from .gaussians import PARAM_NAMES
    tails = {"positions": (3,), "log_scales": (3,), "rotations": (4,), "opacity_logits": (),
             "sh_coeffs": ((degree + 1) ** 2, 3)}
    n = rows.shape[0]
    off = 0
    groups = []
    for _ in range(3):
        g = {}
        for k in PARAM_NAMES:
            wd = _param_width(k, degree)
            g[k] = rows[:, off:off + wd].reshape((n,) + tails[k]).contiguous()
            off += wd
        groups.append(g)
    return groups


def densify_exchange(rs, comm: "TorchComm", it: int, grad_threshold: float,
                     split_threshold: float) -> tuple:
    """Phases 1-3 over a process group: (this rank's new rows in new-id
    order, the new shard map)."""
    payload, counts = densify_local(rs, it, grad_threshold, split_threshold)
    dev = payload.device
    mine = torch.tensor(counts, dtype=torch.int64, device=dev)
    allc = [torch.empty_like(mine) for _ in range(comm.world)]
    comm.dist.all_gather(allc, mine, group=comm.group)
    counts_all = [tuple(int(x) for x in c.tolist()) for c in allc]
    new_ids, smap, send_counts = densify_targets(counts_all, comm.rank, comm.world)
    recv, _ = comm.alltoallv(payload, send_counts)
    recv_ids, _ = comm.alltoallv(torch.from_numpy(new_ids).to(dev), send_counts)
    return assemble_rows(recv, recv_ids, smap, comm.rank), smap


def _rank_from_rows(rs: "RankStep", rows: torch.Tensor, smap: ShardMap) -> "RankStep":
    """New RankStep for this rank from its rows in new-id order."""
    deg = rs.cloud.degree
    groups = unpack_rows(rows, deg)
    new = RankStep(rs.rank, rs.world, smap, rs.part, groups[0], deg, rs.cfg, rs.scene_extent,
                   rs.dev, rs.cfg.background)
    new.m, new.v = groups[1], groups[2]
    return new


def densify_thresholds(cfg, width: int, scene_extent: float) -> tuple:
    from .densify import SPLIT_EXTENT_FRACTION
    res = cfg.resolution if cfg.resolution is not None else width
    return (cfg.effective_grad_threshold(res),
            cfg.split_threshold if cfg.split_threshold is not None
            else SPLIT_EXTENT_FRACTION * scene_extent)


def densify_due(cfg, it: int) -> bool:
    return (cfg.densify and cfg.densify_start <= it <= cfg.effective_densify_stop()
            and it % cfg.densify_interval == 0)


def comm_densify(rs: "RankStep", comm: "TorchComm", it: int) -> "RankStep":
    """Densify + rebalance on this rank (multi-process): one all_gather of the
    class counts, then two all-to-all-v (row payloads, new ids)."""
    gt, st = densify_thresholds(rs.cfg, rs.W, rs.scene_extent)
    rows, smap = densify_exchange(rs, comm, it, gt, st)
    return _rank_from_rows(rs, rows, smap)


def emulated_densify(ranks: list, it: int) -> list:
    """The same three phases for W ranks in sequence on one GPU."""
    W = len(ranks)
    gt, st = densify_thresholds(ranks[0].cfg, ranks[0].W, ranks[0].scene_extent)
    outs = [densify_local(r, it, gt, st) for r in ranks]
    counts_all = [o[1] for o in outs]
    plans = [densify_targets(counts_all, w, W) for w in range(W)]
    smap = plans[0][1]
    new_ranks = []
    for dst in range(W):
        parts, ids = [], []
        for src in range(W):
            sc = plans[src][2]
            o = sum(sc[:dst])
            parts.append(outs[src][0][o:o + sc[dst]])
            ids.append(torch.from_numpy(plans[src][0][o:o + sc[dst]]))
        rows = assemble_rows(torch.cat(parts, 0), torch.cat(ids, 0).to(ranks[dst].dev), smap,
                             dst)
        new_ranks.append(_rank_from_rows(ranks[dst], rows, smap))
    return new_ranks


# ------------------------------------------------------------------ drivers --

def comm_step(rs: RankStep, comm: TorchComm, cam, gt: torch.Tensor, it: int,
              timer=None) -> torch.Tensor:
    """One iteration on this rank (multi-process, one GPU per rank).  timer:
    optional engine.PhaseTimer (CUDA events between the phases)."""
    from .engine import _mark
    _mark(timer, "begin")
    rec, cnt = rs.phase_project(cam)
    _mark(timer, "project_route")
    rrec, _ = comm.alltoallv(rec, cnt)
    _mark(timer, "a2a_splats")
    to_prev, to_next = rs.phase_render(rrec)
    _mark(timer, "bin_render")
    sp, sn = rs.halo_shapes()
    got_prev, got_next = comm.halo(to_prev, to_next, sp, sn, torch.float32, rs.dev)
    _mark(timer, "halo")
    parts = rs.phase_loss(got_prev, got_next, gt)
    comm.allreduce_sum_(parts)
    loss = rs.finish_loss()
    _mark(timer, "loss_allreduce")
    grec, gcnt = rs.phase_backward(timer)
    _mark(timer, "block_fold")
    rg, _ = comm.alltoallv(grec, gcnt)
    _mark(timer, "a2a_grads")
    rs.phase_update(rg, it)
    _mark(timer, "owner_fold_chain_adam")
    return loss


def comm_pair_counts(rs: RankStep, comm: TorchComm, cam) -> dict:
    """Roofline units of this rank's band for view `cam`: pairs
    iterated (I_f), contributing (C) and the backward's I_b (sum of the
    last-contributor index) over the reference's full lists; no state change."""
    rec, cnt = rs.phase_project(cam)
    rrec, _ = comm.alltoallv(rec, cnt)
    rs.phase_render(rrec, count=True)
    px = (rs.prow1 - rs.prow0) * rs.W
    out = {"M": rs.M, "E": rs.E, "P": px,
           "I_f": int(rs.n_iter[:px].sum(dtype=torch.int64)),
           "C": int(rs.n_contrib[:px].sum(dtype=torch.int64)),
           "I_b": int(rs.n_last[:px].sum(dtype=torch.int64))}
    rs.n_contrib = rs.n_iter = None
    return out


def emulated_step(ranks: list, cam, gt: torch.Tensor, it: int) -> torch.Tensor:
    """The same phases for W ranks executed in sequence on ONE GPU with the
    exchanges done by in-process copies (no kernel waits on another rank).
    Used to check bitwise W-invariance on a single B200."""
    W = len(ranks)
    sent = [r.phase_project(cam) for r in ranks]

    def exchange(sent_lists):
        out = []
        for dst in range(W):
            parts = []
            for src in range(W):
                rec, cnt = sent_lists[src]
                o = sum(cnt[:dst])
                parts.append(rec[o:o + cnt[dst]])
            out.append(torch.cat(parts, 0) if parts else None)
        return out

    recv = exchange(sent)
    bounds = [r.phase_render(recv[i]) for i, r in enumerate(ranks)]
    for i, r in enumerate(ranks):
        got_prev = bounds[i - 1][1] if i > 0 else None
        got_next = bounds[i + 1][0] if i + 1 < W else None
        r.phase_loss(got_prev, got_next, gt)
    total = torch.zeros_like(ranks[0].parts)
    for r in ranks:
        total += r.parts
    for r in ranks:
        r.parts.copy_(total)
    loss = ranks[0].finish_loss()
    grads = [r.phase_backward() for r in ranks]
    grecv = exchange(grads)
    for i, r in enumerate(ranks):
        r.phase_update(grecv[i], it)
    return loss


def make_ranks(cloud, width, height, config, scene_extent, workers, device,
               canon_rows=CANON_ROWS, only_rank=None) -> tuple:
    """Shard `cloud` (device tensors) over `workers` ranks; returns (ranks,
    shard map, pixel partition).  only_rank builds just that rank's state."""
    from .gaussians import PARAM_NAMES
    smap = partition_gaussians(cloud.count, workers)
    part = partition_pixels(width, height, TILE, workers, canon_rows)
    starts = smap.starts
    ranks = []
    for w in range(workers):
        if only_rank is not None and w != only_rank:
            continue
        params = {k: getattr(cloud, k)[starts[w]:starts[w + 1]].contiguous().clone()
                  for k in PARAM_NAMES}
        ranks.append(RankStep(w, workers, smap, part, params, cloud.degree, config, scene_extent,
                              device, config.background))
    return ranks, smap, part


def gather_cloud(ranks: list):
    """Concatenate the shards in global id order (engine.py:564-590)."""
    from .gaussians import GaussianCloud, PARAM_NAMES
    return GaussianCloud(*(torch.cat([getattr(r.cloud, k) for r in ranks], 0) for k in PARAM_NAMES),
                         degree=ranks[0].cloud.degree)


def run_training_distributed(dataset, config, workers: int, init_cloud=None, evaluate=True):
    """Sharded training under torch.distributed (one process per GPU, launched
    with torchrun, WORLD_SIZE == workers).  Rank 0 returns (cloud, report)."""
    import torch.distributed as dist
    from .engine import Trainer, _images_to_device
    from .gaussians import cloud_from_points, to_device_cloud
    from .training import TrainReport, build_schedule, init_log_scales
    if not dist.is_initialized():
        raise RuntimeError("workers > 1 needs torch.distributed (launch with torchrun, one "
                           "process per GPU)")
    comm = TorchComm()
    if comm.world != workers:
        raise ValueError(f"workers={workers} but WORLD_SIZE={comm.world}")
    dev = L.require_cuda()
    if init_cloud is None:
        pts = np.asarray(dataset.points.positions, dtype=np.float64)
        cloud = cloud_from_points(pts, init_log_scales(pts), config.sh_degree, dev)
    else:
        cloud = to_device_cloud(init_cloud, dev, torch.float32)
    (rs,), smap, part = make_ranks(cloud, dataset.width, dataset.height, config,
                                   dataset.scene_extent, workers, dev, only_rank=comm.rank)
    images = _images_to_device(dataset.images, dev)
    schedule = build_schedule(config.iterations, dataset.view_count, config.seed)
    losses = torch.zeros(max(config.iterations, 1), dtype=torch.float64, device=dev)
    wall = 0.0
    for it in range(1, config.iterations + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        v = schedule[it - 1]
        loss = comm_step(rs, comm, dataset.cameras[v], images[v], it)
        losses[it - 1] = loss[0]
        if densify_due(config, it):
            rs = comm_densify(rs, comm, it)
            smap = partition_gaussians(sum(_all_sizes(rs, comm)), workers)
        torch.cuda.synchronize()
        wall += time.perf_counter() - t0
    # gather the shards on rank 0 (checkpoint gather, engine.py:564-590)
    from .gaussians import PARAM_NAMES
    full = {}
    for k in PARAM_NAMES:
        t = getattr(rs.cloud, k)
        sizes = smap.sizes
        bufs = [torch.empty((sizes[w],) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
                for w in range(workers)]
        dist.all_gather(bufs, t.contiguous())
        full[k] = torch.cat(bufs, 0)
    from .gaussians import GaussianCloud
    result = GaussianCloud(*(full[k] for k in PARAM_NAMES), degree=rs.cloud.degree)
    report = TrainReport(workers=workers, resolution=config.resolution or dataset.width)
    report.iteration_losses = [float(x) for x in losses[:config.iterations].tolist()]
    report.total_wall_s = wall
    if evaluate and comm.rank == 0:
        tr = Trainer(result, dataset.width, dataset.height, config, dataset.scene_extent, dev)
        report.records.append(tr.evaluate(dataset.cameras, images, config.iterations, wall))
    return result, report


def _all_sizes(rs: "RankStep", comm: "TorchComm") -> list:
    mine = torch.tensor([rs.n], dtype=torch.int64, device=rs.dev)
    allc = [torch.empty_like(mine) for _ in range(comm.world)]
    comm.dist.all_gather(allc, mine, group=comm.group)
    return [int(c.item()) for c in allc]
