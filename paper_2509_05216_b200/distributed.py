"""Sharded multi-GPU training step (reference distributed.py + engine.py W>1).

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  Each GPU
owns a contiguous shard of Gaussians (partition_gaussians, distributed.py:
72-88) and a contiguous ROW BAND of image tiles (partition_pixels; the
reference's round-robin tiles ship 2.3x more splat records at 8 GPUs, SURVEY
§8e).  One iteration, per rank, is a fixed sequence of phases separated by
collectives -- the reference's barrier-separated phases (engine.py:184-537):

  plan      isg_preprocess on the shard; isg_route_plan: per destination band
            the shard's splat records, canonical-block gradient records and
            tile entries                      -> counts all-to-all (3 x W int64)
  sizes     the iteration's ONE host synchronisation: every buffer size and
            exchange split of the step
  pack      isg_route_pack: key + 64 B payload per (splat, band), in shard row
            order per band; the own band's straight into the receive buffers
                                              -> point-to-point group #1
  render    depth sort of the received splats (receive order = global id
            order), band tile lists, raster forward into a window buffer
                                              -> halo rows
  loss      isg_loss_rows on the band (+16/+10 halo rows); block partials of
            the loss                          -> all-reduce
  backward  raster backward on the band, per-(splat, canonical block) fold
            into records by receive index     -> point-to-point group #2
  update    owner fold through the route plan (bands ascending, no sort),
            chain rule + stats + Adam on the shard

Every cross-GPU meeting point has a canonical order (global (depth, id) sort;
canonical 8-tile-row blocks summed in band order; fixed-order loss sums), so
the result is bitwise identical for any GPU count (tests/test_dist_gpu.py
checks W = 1..8 against the single-GPU engine on one B200 by running the
ranks' phases in sequence with an in-process exchange, up to config 3).

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
CANON_ROWS = 2
# our kernels per sharded step at config 3 (every launch is ours; counted
# from the code path, as the single-GPU count is from its ncu launch list):
# preprocess, route plan + scan, pack, depth radix sort (5 passes x 3 + tie
# fix), band binning with live counts (gather + 2 scans x 2), live emission,
# tile radix sort (2 x 3), offsets, heavy-first order (1), raster fwd, loss
# (3) + band cost, raster bwd, band blocks + scan (2), band fold, owner
# fold, chain, Adam.  The exchange barriers / halo copies / NCCL collectives
# and memsets are not counted.
LAUNCHES_PER_STEP = 47


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
        wts = np.asarray(weights, dtype=np.float64)
        if wts.shape != (n_blocks,):
            raise ValueError(f"weights: {wts.shape} != ({n_blocks},) canonical blocks")
        cuts = minmax_cuts(wts, workers)
    band_rows = [min(c * canon_rows, tiles_y) for c in cuts]
    return PixelPartition(width, height, tile_size, workers, tiles_x, tiles_y, band_rows,
                          canon_rows)


def minmax_cuts(weights: np.ndarray, parts: int) -> list:
    """Contiguous cut of `weights` into `parts` non-empty groups that
    minimises the largest group sum (exact DP over the cut positions, ties to
    the earliest cut); cuts[0] = 0, cuts[parts] = len(weights)."""
    w = np.asarray(weights, dtype=np.float64)
    b = w.shape[0]
    pre = np.concatenate([[0.0], np.cumsum(w)])
    seg = pre[None, :] - pre[:, None]          # seg[i, j] = sum of w[i:j]
    invalid = np.tril(np.ones((b + 1, b + 1), dtype=bool))  # j <= i: empty group
    dp = np.full(b + 1, np.inf)
    dp[0] = 0.0
    args = []
    for _ in range(parts):
        m = np.maximum(dp[:, None], seg)
        m[invalid] = np.inf
        args.append(np.argmin(m, axis=0))
        dp = m[args[-1], np.arange(b + 1)]
    cuts = [b]
    for a in reversed(args):
        cuts.append(int(a[cuts[-1]]))
    return cuts[::-1]


def band_cost_ratio(weights: np.ndarray, band_rows: list, canon_rows: int) -> float:
    """max / mean of the per-band sums of per-block costs."""
    w = np.asarray(weights, dtype=np.float64)
    sums = np.array([w[band_rows[k] // canon_rows:(band_rows[k + 1] + canon_rows - 1)
                      // canon_rows].sum() for k in range(len(band_rows) - 1)])
    return float(sums.max() / max(sums.mean(), 1e-300))


def route_rows(tile_min, tile_max, part_or_workers, tiles_x: int | None = None):
    """(n, W) u8 membership mask of rows over workers.

    route_rows(tile_min, tile_max, workers, tiles_x): the reference's
    round-robin routing (distributed.py:127-136): row i reaches worker w iff
    its tile rect touches a tile whose linear id is congruent to w, on the
    device (isg_route_mask); returns a device tensor.
    route_rows(tile_min, tile_max, part): a PixelPartition of row bands: row i
    reaches worker w iff its rect's tile rows overlap w's band (numpy)."""
    if isinstance(part_or_workers, PixelPartition):
        part = part_or_workers
        tmin = np.asarray(tile_min.cpu() if isinstance(tile_min, torch.Tensor) else tile_min)
        tmax = np.asarray(tile_max.cpu() if isinstance(tile_max, torch.Tensor) else tile_max)
        n = tmin.shape[0]
        mask = np.zeros((n, part.workers), dtype=np.uint8)
        for w in range(part.workers):
            lo, hi = part.band_rows[w], part.band_rows[w + 1]
            mask[:, w] = ((tmin[:, 1] < hi) & (tmax[:, 1] >= lo)).astype(np.uint8)
        return mask
    workers = int(part_or_workers)
    if tiles_x is None:
        raise ValueError("route_rows(tile_min, tile_max, workers, tiles_x) needs tiles_x")
    if workers < 1 or workers > 64:
        raise ValueError("workers must be in 1..64")
    dev = L.require_cuda()

    def dev_i32(a):
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
        return t.to(device=dev, dtype=torch.int32).reshape(-1, 2)

    rects = torch.cat([dev_i32(tile_min), dev_i32(tile_max)], 1).contiguous()
    n = rects.shape[0]
    mask = torch.zeros((n, workers), dtype=torch.uint8, device=dev)
    L.check(L.lib().isg_route_mask(n, L.ptr(rects), int(tiles_x), workers, L.ptr(mask),
                                   L.stream_ptr()), "isg_route_mask")
    return mask


def route_splats(splats, part) -> list:
    """Per-destination splat lists, each in (depth, index) order
    (distributed.py:139-154): a splat goes to every worker owning a tile of
    its tile span (part.assignment: round-robin tiles or row bands)."""
    assign = np.asarray(part.assignment)
    out = [[] for _ in range(part.workers)]
    for s in sorted(splats, key=lambda s: (s.depth, s.gaussian_index)):
        (x0, y0), (x1, y1) = s.tile_span
        owners = np.unique(assign[(np.arange(y0, y1 + 1)[:, None] * part.tiles_x
                                   + np.arange(x0, x1 + 1)[None, :]).ravel()])
        for d in owners.tolist():
            out[d].append(s)
    return out


def rebalance(shard_map: ShardMap, counts: list) -> tuple:
    """Migration plan that evens the shard sizes to within one row
    (distributed.py:229-268): every over-full shard gives up its lowest-id
    excess rows; the pooled rows, taken in ascending id, fill the under-full
    shards in worker order.  Returns ((gaussian, from, to) moves in ascending
    id within each destination, the resulting ShardMap)."""
    if list(counts) != shard_map.sizes:
        raise ValueError("counts disagree with the shard map")
    w, n = shard_map.workers, shard_map.total
    q, r = divmod(n, w)
    target = [q + int(k < r) for k in range(w)]
    sizes = shard_map.sizes
    donated = sorted((int(g), src) for src in range(w)
                     for g in shard_map.lists[src][:max(sizes[src] - target[src], 0)])
    plan, it = [], iter(donated)
    for dst in range(w):
        for _ in range(max(target[dst] - sizes[dst], 0)):
            g, src = next(it)
            plan.append((g, src, dst))
    leaving = {g for g, _, _ in plan}
    arriving = [[] for _ in range(w)]
    for g, _, dst in plan:
        arriving[dst].append(g)
    lists = [np.sort(np.concatenate([shard_map.lists[u][~np.isin(shard_map.lists[u],
                                                                   list(leaving))],
                                     np.asarray(arriving[u], dtype=np.int64)])).astype(np.int64)
             for u in range(w)]
    return plan, ShardMap.from_lists(lists, n)


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

    def __init__(self, group=None, peers: bool = False, height: int = 0, width: int = 0,
                 device=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        # peer-store exchange (PeerBuffers over symmetric memory) instead of
        # point-to-point copies for the splat records, halo and gradients
        self.peers = PeerBuffers(self.world, height, width, device, group) if peers else None

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

    def counts(self, mine: torch.Tensor, out: torch.Tensor) -> None:
        """(W, 3) per-band counts of this shard -> out (W, W, 3), out[s] =
        shard s's row (one all-gather of 3 int64 per pair, on the device):
        every rank sees the whole count matrix, so every rank can place its
        records directly in every other rank's buffers (peer exchange)."""
        self.dist.all_gather_into_tensor(out.view(-1, *mine.shape[1:]), mine.contiguous(),
                                         group=self.group)

    def exchange(self, ops: list) -> None:
        """Point-to-point segments: ops = [(peer, [send tensors], [recv
        tensors])], the same tensor count per peer on both sides; one NCCL
        group (batch_isend_irecv).  Empty segments are skipped."""
        P2POp = self.dist.P2POp
        p2p = []
        for peer, sends, recvs in ops:
            for t in recvs:
                if t.numel():
                    p2p.append(P2POp(self.dist.irecv, t, peer, self.group))
            for t in sends:
                if t.numel():
                    p2p.append(P2POp(self.dist.isend, t, peer, self.group))
        if p2p:
            for req in self.dist.batch_isend_irecv(p2p):
                req.wait()

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


# ------------------------------------------------------- exchange layout --

def exchange_layout(mat: np.ndarray, me: int) -> dict:
    """Where every record of the iteration lives, from the all-gathered count
    matrix mat (W, W, 3): mat[s, d] = shard s's (splat records, canonical
    block records, tile entries) for band d.  Band d receives splat records
    in source order, so shard me's segment starts at pack_at[d]; owner s
    receives block records in band order, so band me's segment for owner s
    starts at grad_at[s], and band b's segment of this rank's own receive
    buffer at grad_seg[b].  need_r / need_g: the largest receive counts over
    the ranks (the capacity of the peer buffers, the same on every rank)."""
    mat = np.asarray(mat, dtype=np.int64)
    rec, blk = mat[:, :, 0], mat[:, :, 1]
    W = mat.shape[0]
    return {
        "pack_at": [int(rec[:me, d].sum()) for d in range(W)],
        "grad_at": [int(blk[s, :me].sum()) for s in range(W)],
        "grad_seg": [int(v) for v in np.concatenate([[0], np.cumsum(blk[me])])],
        "need_r": int(rec.sum(axis=0).max()) if W else 0,
        "need_g": int(blk.sum(axis=1).max()) if W else 0,
    }


class PeerBuffers:
    """The peer-store exchange's receive buffers: every rank's
    splat-record receive buffers (depth keys, 64-byte payloads), gradient
    receive buffer and band image window live in torch symmetric memory, so
    each rank maps every peer's buffers over NVLink and the producing kernels
    store into them directly: the pack kernel writes each band's records into
    that band's GPU (isg_route_pack_peer), the band fold writes each block
    record into its owner's GPU (isg_band_fold_peer), the forward's boundary
    rows go straight into the neighbours' windows.  A barrier (a signal-pad
    kernel on the stream) follows each of the three; nothing is staged or
    copied by NCCL.  The capacity is the max over the ranks of the receive
    counts (exchange_layout), so every rank makes the same (collective)
    growth decision."""

    SLACK = 1.25

    def __init__(self, world: int, height: int, width: int, device, group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        self.symm = symm
        self.group = group if group is not None else dist.group.WORLD
        self.world = world
        self.H, self.W = height, width
        self.dev = device
        self.win = symm.empty(height * width * 3, dtype=torch.float32, device=device)
        self.win.zero_()
        self.win_h = symm.rendezvous(self.win, self.group)
        self.win_ptrs = list(self.win_h.buffer_ptrs)
        self.cap_r = self.cap_g = 0
        self.buf = self.h = None
        self.ptrs = [0] * world
        # a first buffer now, so a box without peer mappings fails here (where
        # the caller can fall back to the point-to-point exchange), not mid-step
        self.ensure(1 << 16, 1 << 16)
        self.barrier()

    def ensure(self, need_r: int, need_g: int) -> None:
        if need_r <= self.cap_r and need_g <= self.cap_g and self.buf is not None:
            return
        cap_r = max(self.cap_r, int(need_r * self.SLACK) + 16)
        cap_r += cap_r & 1                      # payloads 16-byte aligned
        cap_g = max(self.cap_g, int(need_g * self.SLACK) + 16)
        self.buf = self.h = None
        self.buf = self.symm.empty(72 * cap_r + 72 * cap_g, dtype=torch.uint8, device=self.dev)
        self.h = self.symm.rendezvous(self.buf, self.group)
        self.ptrs = list(self.h.buffer_ptrs)
        self.cap_r, self.cap_g = cap_r, cap_g

    def bind(self, rs: "RankStep") -> None:
        cr, cg = self.cap_r, self.cap_g
        b = self.buf
        rs.keys_recv = b[:8 * cr].view(torch.int64)
        rs.pay_recv = b[8 * cr:72 * cr].view(torch.int32).view(cr, 16)
        rs.grad_recv = b[72 * cr:72 * cr + 72 * cg].view(torch.float64).view(cg, 9)
        rs.window = self.win.view(self.H, self.W, 3)

    def keys_ptr(self, d: int) -> int:
        return self.ptrs[d]

    def pay_ptr(self, d: int) -> int:
        return self.ptrs[d] + 8 * self.cap_r

    def grad_ptr(self, d: int) -> int:
        return self.ptrs[d] + 72 * self.cap_r

    def window_ptr(self, d: int) -> int:
        return self.win_ptrs[d]

    def barrier(self) -> None:
        self.win_h.barrier(channel=0)


class EmulatedPeers:
    """The same peer-store layout for W ranks held by one process on one GPU
    (emulated_step): the 'peer' pointers are the other rank objects' own
    buffers, and the phases run rank after rank, so no barrier is needed."""

    def __init__(self, ranks: list):
        self.ranks = ranks

    def ensure(self, need_r: int, need_g: int) -> None:
        for r in self.ranks:
            r.keys_recv = _grow(r.keys_recv, need_r, dtype=torch.int64, device=r.dev)
            r.pay_recv = _grow(r.pay_recv, need_r, (16,), dtype=torch.int32, device=r.dev)
            r.grad_recv = _grow(r.grad_recv, need_g, (9,), dtype=torch.float64, device=r.dev)

    def bind(self, rs: "RankStep") -> None:
        pass

    def keys_ptr(self, d: int) -> int:
        return self.ranks[d].keys_recv.data_ptr()

    def pay_ptr(self, d: int) -> int:
        return self.ranks[d].pay_recv.data_ptr()

    def grad_ptr(self, d: int) -> int:
        return self.ranks[d].grad_recv.data_ptr()

    def window_ptr(self, d: int) -> int:
        return self.ranks[d].window.data_ptr()

    def barrier(self) -> None:
        pass


# --------------------------------------------------------------- rank state --

def _grow(buf, n: int, tail=(), dtype=torch.float32, device=None, slack: float = 1.25):
    """Capacity-managed buffer: reallocated only when `n` rows do not fit."""
    if buf is None or buf.shape[0] < n:
        return torch.empty((max(int(n * slack), 16),) + tuple(tail), dtype=dtype, device=device)
    return buf


class RankStep:
    """One rank's shard, band and buffers, with the phases of an iteration.

    Per iteration there is exactly ONE host synchronisation (phase_sizes):
    after the route plan, every rank knows per destination band the number of
    splat records, canonical-block gradient records and tile entries its
    shard produces; one all-to-all of those 3 x W counts and one 48 x W-byte
    read give every size of the iteration (receive counts, the band's tile
    entries, both directions of the gradient exchange).  Records of the
    rank's own band are written straight into its receive buffers (no self
    copy); gradient records are laid out by receive index, so the segment for
    each owner is already in its shard row order and the owner folds them
    through its route plan with no sort."""

    def __init__(self, rank: int, world: int, shards: ShardMap, part: PixelPartition,
                 params: dict, degree: int, config, scene_extent: float, device,
                 background=(1.0, 1.0, 1.0)):
        from .gaussians import GaussianCloud, PARAM_NAMES
        self.rank, self.world = rank, world
        self.dev = device
        self.cfg = config
        self.scene_extent = float(scene_extent)
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
        self.image_tiles = part.tiles_x * part.tiles_y  # the chunk policy: per image, not band
        self.bg = (ctypes.c_double * 3)(*[float(v) for v in background])
        d = device
        n = self.n
        # shard-side buffers
        self.key = torch.empty(n, dtype=torch.int64, device=d)
        self.rect = torch.empty((n, 4), dtype=torch.int32, device=d)
        self.feat = torch.empty((n, 12), dtype=torch.float32, device=d)
        self.flag = torch.empty(n, dtype=torch.uint8, device=d)
        self.grad2d = torch.zeros((n, 9), dtype=torch.float64, device=d)
        pe = ctypes.c_int64(0)
        L.check(L.lib().isg_route_plan_size(n, world, ctypes.byref(pe)), "route plan size")
        self.plan = torch.empty(max(pe.value, 1), dtype=torch.int64, device=d)
        # counts = this shard's per-band totals; cmat[s] = shard s's (all-gathered)
        self.counts = torch.zeros((world, 3), dtype=torch.int64, device=d)
        self.cmat = torch.zeros((world, world, 3), dtype=torch.int64, device=d)
        self.cmat_host = torch.zeros((world, world, 3), dtype=torch.int64).pin_memory()
        # peer-store exchange (PeerBuffers / EmulatedPeers) or None: point-to-point copies
        self.peers = None
        # (M, E, live E) of the band's binning; only the live count is read (on the device)
        self.bin_counts = torch.zeros(3, dtype=torch.int64, device=d)
        nf = ctypes.c_int32(0)
        na = ctypes.c_int32(0)
        L.lib().isg_loss_partials_size(self.H, self.W, ctypes.byref(nf), ctypes.byref(na))
        self.n_ps, self.n_pl = nf.value, na.value
        self.loss_dev = torch.zeros(1, dtype=torch.float64, device=d)
        self.ws = [L.Workspace() for _ in range(4)]
        # receive-side / band buffers (grown on demand)
        self.keys_recv = self.pay_recv = self.keys_send = self.pay_send = None
        self.vals0 = self.key_sorted = self.order = None
        self.rect_sorted = self.feat_sorted = self.emit_off = None
        self.tk = self.tv = self.tk_sorted = self.entries = self.partials = None
        self.live_off = self.live_mask = self.slot_rank = self.iota = None
        self.live = False
        self.cmask = self.nb = self.gpos = self.gbuf = self.grad_recv = None
        self.to_keys = self.to_vals = self.to_keys_s = self.to_order = self.tile_order = None
        self.chunks = None
        import os
        self.heavy_first = os.environ.get("ISOGS_HEAVY_FIRST", "1") != "0"
        # band-side image buffers at full-image size: bands move when the
        # partition is rebalanced, the buffers do not
        self.window = torch.zeros((self.H, self.W, 3), dtype=torch.float32, device=d)
        self.t_final = torch.empty(self.H * self.W, dtype=torch.float32, device=d)
        self.n_last = torch.empty(self.H * self.W, dtype=torch.int32, device=d)
        self.dl = torch.empty((self.H * self.W, 3), dtype=torch.float32, device=d)
        # load balance: per-canonical-block raster cost (all-reduced with the
        # loss partials), its moving average, re-cut every REBALANCE_EVERY steps
        self.n_blk = (part.tiles_y + part.canon_rows - 1) // part.canon_rows
        self.parts = torch.zeros(self.n_ps + self.n_pl + self.n_blk, dtype=torch.float64,
                                 device=d)
        self.cost_host = torch.zeros(self.n_blk, dtype=torch.float64).pin_memory()
        self.cost_ema = None
        self.pending_part = None
        self.balance = {"recuts": 0, "ratio_equal": None, "ratio_now": None}
        self.set_partition(part)

    def set_partition(self, part: PixelPartition) -> None:
        """Adopt a (new) row-band partition; results do not depend on it."""
        self.part = part
        rank = self.rank
        self.trow0, self.trow1 = part.band_rows[rank], part.band_rows[rank + 1]
        self.prow0, self.prow1 = part.pixel_rows(rank)
        self.win0 = max(0, self.prow0 - 16)
        self.win1 = min(self.H, self.prow1 + 10)
        self.band_host = (ctypes.c_int32 * (self.world + 1))(*part.band_rows)
        self.n_tiles = (self.trow1 - self.trow0) * self.tiles_x
        self.tile_bits = _bits(self.n_tiles)
        self.offsets = torch.empty(self.n_tiles + 1, dtype=torch.int32, device=self.dev)

    def _vptr(self, t: torch.Tensor, row0: int, row_elems: int) -> int:
        """Virtual base pointer so that global row `row0` maps to t's start."""
        return t.data_ptr() - row0 * row_elems * t.element_size()

    # -- phase 1: project + route plan ------------------------------------
    def phase_plan(self, cam) -> torch.Tensor:
        """Preprocess the shard and plan its records per band; returns the
        (W, 3) per-band totals (splat records, block records, tile entries)
        to exchange."""
        lib, s = L.lib(), L.stream_ptr()
        if self.pending_part is not None:
            self.set_partition(self.pending_part)
            self.pending_part = None
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
        L.check(lib.isg_route_plan(self.n, L.ptr(self.flag), L.ptr(self.rect), self.band_host,
                                   self.world, self.part.canon_rows, L.ptr(self.plan),
                                   L.ptr(self.counts), s), "isg_route_plan")
        return self.counts

    # -- the one host synchronisation --------------------------------------
    def phase_sizes(self) -> None:
        """Read the count matrix (cmat, filled by the counts all-gather) and
        size the iteration."""
        self.cmat_host.copy_(self.cmat, non_blocking=True)
        # the previous step's all-reduced band costs ride on the same sync
        self.cost_host.copy_(self.parts[self.n_ps + self.n_pl:], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        h = self.cmat_host.numpy()
        W, me = self.world, self.rank
        mine, recv = h[me], h[:, me]
        self.lay = exchange_layout(h, me)
        if self.peers is not None:
            self.peers.ensure(self.lay["need_r"], self.lay["need_g"])
        self.send_cnt = [int(x) for x in mine[:, 0]]
        self.recv_cnt = [int(x) for x in recv[:, 0]]
        self.gsend_cnt = [int(x) for x in recv[:, 1]]   # band -> owner s
        self.grecv_cnt = [int(x) for x in mine[:, 1]]   # owner <- band d
        self.R = sum(self.recv_cnt)
        self.E = int(recv[:, 2].sum())
        self.NR = sum(self.gsend_cnt)
        self.recv_off = np.concatenate([[0], np.cumsum(self.recv_cnt)]).astype(np.int64)
        self.gpos_off = np.concatenate([[0], np.cumsum(self.gsend_cnt)]).astype(np.int64)
        others = [c if d != me else 0 for d, c in enumerate(self.send_cnt)]
        self.send_off = np.concatenate([[0], np.cumsum(others)]).astype(np.int64)
        gothers = [c if d != me else 0 for d, c in enumerate(self.grecv_cnt)]
        self.grecv_off = np.concatenate([[0], np.cumsum(gothers)]).astype(np.int64)

    # -- phase 2: pack splat records ----------------------------------------
    def phase_pack(self) -> list:
        """Splat records into the send buffers (own band: receive buffers).
        Returns the exchange list [(peer, send tensors, recv tensors)]."""
        lib, s, d = L.lib(), L.stream_ptr(), self.dev
        me = self.rank
        if self.peers is not None:
            # peer-store exchange: each band's segment straight into its GPU
            P, at, W = self.peers, self.lay["pack_at"], self.world
            P.bind(self)
            keys = (ctypes.c_void_p * W)(*[P.keys_ptr(k) + 8 * at[k] for k in range(W)])
            pays = (ctypes.c_void_p * W)(*[P.pay_ptr(k) + 64 * at[k] for k in range(W)])
            if self.n:
                L.check(lib.isg_route_pack_peer(self.n, L.ptr(self.flag), L.ptr(self.rect),
                                                L.ptr(self.key), L.ptr(self.feat), self.band_host,
                                                W, L.ptr(self.plan), keys, pays, s),
                        "isg_route_pack_peer")
            return []
        R, S = self.R, int(self.send_off[-1])
        self.keys_recv = _grow(self.keys_recv, R, dtype=torch.int64, device=d)
        self.pay_recv = _grow(self.pay_recv, R, (16,), dtype=torch.int32, device=d)
        self.keys_send = _grow(self.keys_send, S, dtype=torch.int64, device=d)
        self.pay_send = _grow(self.pay_send, S, (16,), dtype=torch.int32, device=d)
        dest = (ctypes.c_int64 * self.world)(*[
            int(self.recv_off[me]) if k == me else int(self.send_off[k])
            for k in range(self.world)])
        if self.n:
            L.check(lib.isg_route_pack(self.n, L.ptr(self.flag), L.ptr(self.rect), L.ptr(self.key),
                                       L.ptr(self.feat), self.band_host, self.world,
                                       L.ptr(self.plan), dest, me, L.ptr(self.keys_send),
                                       L.ptr(self.pay_send), L.ptr(self.keys_recv),
                                       L.ptr(self.pay_recv), s), "isg_route_pack")
        ops = []
        for peer in range(self.world):
            if peer == me:
                continue
            a, b = int(self.send_off[peer]), int(self.send_off[peer + 1])
            c0, c1 = int(self.recv_off[peer]), int(self.recv_off[peer + 1])
            ops.append((peer, [self.keys_send[a:b], self.pay_send[a:b]],
                        [self.keys_recv[c0:c1], self.pay_recv[c0:c1]]))
        return ops

    # -- phase 3: render the band -----------------------------------------
    def phase_render(self, count: bool = False):
        """Depth order over the received splats (receive order = global id
        order, so the stable sort is the reference's lexsort), the band's
        tile lists and the forward.  count=True: the reference's full band
        lists and the unmasked forward with per-pixel pair counters (n_contrib,
        n_iter) for the roofline units; leaves no state for a backward."""
        lib, s, d = L.lib(), L.stream_ptr(), self.dev
        R, E = self.R, self.E
        if self.vals0 is None or self.vals0.shape[0] < R:
            self.vals0 = torch.arange(max(int(R * 1.25), 16), dtype=torch.int32, device=d)
        self.key_sorted = _grow(self.key_sorted, R, dtype=torch.int64, device=d)
        self.order = _grow(self.order, R, dtype=torch.int32, device=d)
        L.sort_depth(self.keys_recv[:R], self.vals0[:R], self.ws[0], self.key_sorted[:R],
                     self.order[:R])
        self.rect_sorted = _grow(self.rect_sorted, R, (4,), dtype=torch.int32, device=d)
        self.feat_sorted = _grow(self.feat_sorted, R, (12,), dtype=torch.float32, device=d)
        self.emit_off = _grow(self.emit_off, R + 1, dtype=torch.int64, device=d)
        # band lists: live-only for training (pairs no pixel of their tile can
        # composite have no entry and no subtotal slot; the live count stays on
        # the device -- E, the band's tile entries, bounds it); count mode:
        # the reference's full lists
        live = not count
        self.live = live
        k16 = self.n_tiles <= 65536  # 2-byte tile keys (see engine.Rasterizer.forward)
        kb = 2 if k16 else 4
        sz = ctypes.c_size_t(0)
        if live:
            L.check(lib.isg_bin_count_live(None, ctypes.byref(sz), R, None, None, None, None,
                                           None, self.trow0, self.trow1, None, None, None, None,
                                           None, None, None), "bin size")
        else:
            L.check(lib.isg_bin_count_rows(None, ctypes.byref(sz), R, None, None, None,
                                           self.trow0, self.trow1, None, None, None, None, None),
                    "bin size")
        ws = self.ws[2].get(sz.value, d)
        sz = ctypes.c_size_t(ws.numel())
        if live:
            self.live_off = _grow(self.live_off, R + 1, dtype=torch.int64, device=d)
            self.live_mask = _grow(self.live_mask, R, dtype=torch.int64, device=d)
            L.check(lib.isg_bin_count_live(L.ptr(ws), ctypes.byref(sz), R,
                                           L.ptr(self.key_sorted), L.ptr(self.order), None,
                                           L.ptr(self.pay_recv), None, self.trow0, self.trow1,
                                           L.ptr(self.rect_sorted), L.ptr(self.feat_sorted),
                                           L.ptr(self.emit_off), L.ptr(self.live_off),
                                           L.ptr(self.live_mask), L.ptr(self.bin_counts), s),
                    "isg_bin_count_live")
        else:
            L.check(lib.isg_bin_count_rows(L.ptr(ws), ctypes.byref(sz), R, L.ptr(self.key_sorted),
                                           L.ptr(self.order), L.ptr(self.pay_recv), self.trow0,
                                           self.trow1, L.ptr(self.rect_sorted),
                                           L.ptr(self.feat_sorted), L.ptr(self.emit_off),
                                           L.ptr(self.bin_counts), s), "isg_bin_count_rows")
        self.M = R
        kdt = torch.int16 if k16 else torch.int32
        if self.tk is None or self.tk.dtype != kdt:
            self.tk = self.tk_sorted = None
        self.tk = _grow(self.tk, E, dtype=kdt, device=d)
        self.tv = _grow(self.tv, E, dtype=torch.int32, device=d)
        self.tk_sorted = _grow(self.tk_sorted, E, dtype=kdt, device=d)
        self.entries = _grow(self.entries, E, dtype=torch.int32, device=d)
        self.partials = _grow(self.partials, E, (12,), dtype=torch.float32, device=d)
        n_live = self.bin_counts[2:3]  # live pairs (device)
        if E:
            if live:
                from .engine import _iota
                self.slot_rank = _grow(self.slot_rank, E, dtype=torch.int32, device=d)
                self.iota = _iota(self.iota, E, d)
                L.check(lib.isg_bin_emit_live(R, L.ptr(self.rect_sorted), L.ptr(self.emit_off),
                                              L.ptr(self.live_off), L.ptr(self.live_mask),
                                              L.ptr(self.feat_sorted), self.tiles_x, self.trow0,
                                              self.trow1, L.ptr(self.tk), kb,
                                              L.ptr(self.slot_rank), s), "isg_bin_emit_live")
                vals = self.iota
            else:
                emit = lib.isg_bin_emit16 if k16 else lib.isg_bin_emit
                L.check(emit(R, L.ptr(self.rect_sorted), L.ptr(self.emit_off), self.tiles_x,
                             self.trow0, self.trow1, L.ptr(self.tk), L.ptr(self.tv), s),
                        "isg_bin_emit")
                vals = self.tv
            sz = ctypes.c_size_t(0)
            L.check(lib.isg_sort_pairs_dev(None, ctypes.byref(sz), kb, None, None, None, None, E,
                                           None, 0, self.tile_bits, None), "sort size")
            sws = self.ws[0].get(sz.value, d)
            sz = ctypes.c_size_t(sws.numel())
            L.check(lib.isg_sort_pairs_dev(L.ptr(sws), ctypes.byref(sz), kb, L.ptr(self.tk),
                                           L.ptr(self.tk_sorted), L.ptr(vals),
                                           L.ptr(self.entries), E,
                                           L.ptr(n_live) if live else None, 0, self.tile_bits,
                                           s), "isg_sort_pairs_dev")
        L.check(lib.isg_tile_offsets_dev(E, L.ptr(n_live) if live else None,
                                         L.ptr(self.tk_sorted), kb, self.n_tiles,
                                         L.ptr(self.offsets), s), "isg_tile_offsets_dev")
        from .engine import chunk_setup, heavy_first_order
        self.tile_order = heavy_first_order(self, self.n_tiles, self.offsets)
        self.chunks = None if count else chunk_setup(
            self, self.n_tiles, E, self._vptr(self.window, self.win0, self.W * 3))
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
            self.cmask = _grow(self.cmask, lib.isg_contrib_mask_words(E, self.n_tiles),
                               dtype=torch.int32, device=d)
            L.check(lib.isg_raster_fwd_masked(
                self.W, self.H, self.tiles_x, self.trow0, self.trow1, None, 0,
                L.ptr(self.tile_order),
                L.ptr(self.offsets), L.ptr(self.entries), L.ptr(self.feat_sorted),
                ctypes.cast(self.bg, ctypes.c_void_p),
                self._vptr(self.window, self.win0, W3), L.ISG_F32,
                self._vptr(self.t_final, self.prow0, self.W),
                self._vptr(self.n_last, self.prow0, self.W), None, None, None, L.ptr(self.cmask),
                ctypes.byref(self.chunks) if self.chunks is not None else None,
                L.ptr(self.slot_rank), s), "isg_raster_fwd_masked")
        # boundary rows for the neighbours' SSIM halo
        b0, b1 = self.prow0 - self.win0, self.prow1 - self.win0
        n_prev = min(10, b1 - b0) if self.rank > 0 else 0
        n_next = min(16, b1 - b0) if self.rank + 1 < self.world else 0
        if self.peers is not None:
            # straight into the neighbours' windows (their rows above / below their band)
            row = self.W * 3 * 4
            for nb, g0, cnt in ((self.rank - 1, self.prow0, n_prev),
                                (self.rank + 1, self.prow1 - n_next, n_next)):
                if cnt:
                    w0 = max(0, self.part.pixel_rows(nb)[0] - 16)
                    L.check(lib.isg_copy(self.peers.window_ptr(nb) + (g0 - w0) * row,
                                         self.window.data_ptr() + (g0 - self.win0) * row,
                                         cnt * row, s), "isg_copy")
            return None, None
        to_prev = self.window[b0:b0 + n_prev] if n_prev else None
        to_next = self.window[b1 - n_next:b1] if n_next else None
        return to_prev, to_next

    def halo_shapes(self):
        prev = (self.prow0 - self.win0, self.W, 3) if self.rank > 0 else None
        nxt = (self.win1 - self.prow1, self.W, 3) if self.rank + 1 < self.world else None
        return prev, nxt

    # -- phase 4: loss on the band ----------------------------------------
    def phase_loss(self, from_prev, from_next, gt: torch.Tensor):
        lib, s = L.lib(), L.stream_ptr()
        if from_prev is not None and from_prev.shape[0]:
            self.window[:from_prev.shape[0]].copy_(from_prev)
        if from_next is not None and from_next.shape[0]:
            o = self.prow1 - self.win0
            self.window[o:o + from_next.shape[0]].copy_(from_next)
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
            L.check(lib.isg_band_cost(L.ptr(self.n_last), self.prow0, self.prow1, self.W,
                                      self.part.canon_rows,
                                      self.parts.data_ptr() + 8 * (self.n_ps + self.n_pl), s),
                    "isg_band_cost")
        return self.parts

    def finish_loss(self):
        L.check(L.lib().isg_loss_finish(self.H, self.W, float(self.cfg.lambda_dssim),
                                        L.ptr(self.parts), self.parts.data_ptr() + 8 * self.n_ps,
                                        L.ptr(self.loss_dev), L.stream_ptr()), "isg_loss_finish")
        return self.loss_dev

    # -- phase 5: backward + block records for the owners ------------------
    def phase_backward(self, timer=None) -> list:
        """Raster backward on the band, per-(splat, canonical block) fold into
        records by receive index; returns the exchange list."""
        from .engine import _mark
        lib, s, d = L.lib(), L.stream_ptr(), self.dev
        W3 = self.W * 3
        R, me = self.R, self.rank
        if self.n_tiles and self.E:
            from .engine import chunk_items
            chunk_items(self, self.n_tiles)
            L.check(lib.isg_raster_bwd_masked(
                self.W, self.H, self.tiles_x, self.trow0, self.trow1, None, 0,
                L.ptr(self.tile_order),
                L.ptr(self.offsets), L.ptr(self.entries), L.ptr(self.feat_sorted),
                L.ptr(self.rect_sorted), L.ptr(self.emit_off), ctypes.cast(self.bg, ctypes.c_void_p),
                self._vptr(self.t_final, self.prow0, self.W),
                self._vptr(self.n_last, self.prow0, self.W),
                self._vptr(self.dl, self.prow0, W3), L.ISG_F32, L.ptr(self.partials),
                L.ptr(self.cmask), ctypes.byref(self.chunks) if self.chunks is not None else None,
                L.ptr(self.slot_rank), s), "isg_raster_bwd_masked")
        _mark(timer, "raster_bwd")
        self.nb = _grow(self.nb, R, dtype=torch.int64, device=d)
        self.gpos = _grow(self.gpos, R + 1, dtype=torch.int64, device=d)
        if self.peers is not None:
            # peer-store exchange: each block record straight into its owner's GPU
            P, at, W = self.peers, self.lay["grad_at"], self.world
            if R:
                L.check(lib.isg_band_blocks(R, L.ptr(self.pay_recv), self.trow0, self.trow1,
                                            self.part.canon_rows, L.ptr(self.nb), s),
                        "band blocks")
                _scan_i64(self, R, self.nb, self.gpos)
                ends = (ctypes.c_int64 * W)(*[int(v) for v in self.recv_off[1:]])
                bases = (ctypes.c_void_p * W)(*[
                    P.grad_ptr(k) + 72 * (at[k] - int(self.gpos_off[k])) for k in range(W)])
                L.check(lib.isg_band_fold_peer(R, L.ptr(self.live_off), L.ptr(self.partials),
                                               L.ptr(self.rect_sorted), L.ptr(self.order),
                                               L.ptr(self.gpos), self.trow0, self.trow1,
                                               self.part.canon_rows, 1, W, ends, bases, s),
                        "isg_band_fold_peer")
            return []
        self.gbuf = _grow(self.gbuf, self.NR, (9,), dtype=torch.float64, device=d)
        if R:
            L.check(lib.isg_band_blocks(R, L.ptr(self.pay_recv), self.trow0, self.trow1,
                                        self.part.canon_rows, L.ptr(self.nb), s), "band blocks")
            _scan_i64(self, R, self.nb, self.gpos)
            L.check(lib.isg_band_fold(R, L.ptr(self.live_off), L.ptr(self.partials),
                                      L.ptr(self.rect_sorted), L.ptr(self.order),
                                      L.ptr(self.gpos), self.trow0, self.trow1,
                                      self.part.canon_rows, 1, L.ptr(self.gbuf), s),
                    "isg_band_fold")
        G = int(self.grecv_off[-1])
        self.grad_recv = _grow(self.grad_recv, G, (9,), dtype=torch.float64, device=d)
        ops = []
        for peer in range(self.world):
            if peer == me:
                continue
            a, b = int(self.gpos_off[peer]), int(self.gpos_off[peer + 1])
            c0, c1 = int(self.grecv_off[peer]), int(self.grecv_off[peer + 1])
            ops.append((peer, [self.gbuf[a:b]], [self.grad_recv[c0:c1]]))
        return ops

    REBALANCE_EVERY = 8
    COST_EMA = 0.25

    def rebalance(self) -> None:
        """Host side of the load balance, run after the step's launches are
        issued (it overlaps the GPU): fold the previous step's all-reduced
        per-block costs into a moving average and, every REBALANCE_EVERY
        steps, re-cut the bands (exact min-max cut) for the next step if that
        lowers the predicted max/mean by >= 1 %.  Every rank sees the same
        all-reduced costs, so every rank makes the same cut."""
        if self.world == 1:
            return
        cost = self.cost_host.numpy().astype(np.float64)
        tot = cost.sum()
        if tot <= 0:
            return
        cost = cost / tot
        self.cost_ema = cost if self.cost_ema is None else \
            (1.0 - self.COST_EMA) * self.cost_ema + self.COST_EMA * cost
        p = self.part
        self.balance["ratio_now"] = band_cost_ratio(cost, p.band_rows, p.canon_rows)
        eq = partition_pixels(p.width, p.height, p.tile_size, p.workers, p.canon_rows)
        self.balance["ratio_equal"] = band_cost_ratio(cost, eq.band_rows, p.canon_rows)
        self._steps_seen = getattr(self, "_steps_seen", 0) + 1
        if self._steps_seen % self.REBALANCE_EVERY:
            return
        new = partition_pixels(p.width, p.height, p.tile_size, p.workers, p.canon_rows,
                               weights=self.cost_ema)
        now = band_cost_ratio(self.cost_ema, p.band_rows, p.canon_rows)
        if band_cost_ratio(self.cost_ema, new.band_rows, p.canon_rows) <= 0.99 * now:
            self.pending_part = new
            self.balance["recuts"] += 1

    # -- phase 6: owner fold + chain + Adam -------------------------------
    def phase_update(self, it: int):
        from .engine import update_params
        from .optim import position_lr
        me = self.rank
        segs = []
        for b in range(self.world):
            if self.peers is not None:
                segs.append(self.grad_recv.data_ptr() + 72 * self.lay["grad_seg"][b])
            elif b == me:
                segs.append(self.gbuf.data_ptr() + 72 * int(self.gpos_off[me]))
            else:
                segs.append(self.grad_recv.data_ptr() + 72 * int(self.grecv_off[b]))
        seg = (ctypes.c_void_p * self.world)(*segs)
        if not self.n:
            return
        L.check(L.lib().isg_owner_fold_plan(self.n, L.ptr(self.flag), L.ptr(self.rect),
                                            self.band_host, self.world, self.part.canon_rows,
                                            L.ptr(self.plan), seg, L.ptr(self.grad2d),
                                            L.stream_ptr()), "isg_owner_fold_plan")
        cfg = self.cfg
        lrs = [self.scene_extent * position_lr(cfg.lr_position, it, cfg.iterations,
                                               cfg.lr_position_final),
               cfg.lr_scale, cfg.lr_rotation, cfg.lr_opacity, cfg.lr_sh]
        if getattr(self, "grads", None) is None:
            self.grads = {k: torch.empty_like(v) for k, v in self.m.items()}
        update_params(self.cloud, self.m, self.v, self.grads, self.seen, self.grad_accum,
                      self.flag, self.grad2d, self.cam_struct, lrs, it, self.W, self.H)


def _scan_i64(rs: RankStep, n: int, cnt: torch.Tensor, off: torch.Tensor) -> None:
    lib = L.lib()
    sz = ctypes.c_size_t(0)
    L.check(lib.isg_scan_i64(None, ctypes.byref(sz), n, None, None, None, None), "scan size")
    buf = rs.ws[1].get(sz.value, rs.dev)
    sz = ctypes.c_size_t(buf.numel())
    L.check(lib.isg_scan_i64(L.ptr(buf), ctypes.byref(sz), n, L.ptr(cnt), L.ptr(off), None,
                             L.stream_ptr()), "isg_scan_i64")


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
    """One iteration on this rank (multi-process, one GPU per rank), with one
    host synchronisation (phase_sizes).  timer: optional engine.PhaseTimer
    (CUDA events between the phases)."""
    from .engine import _mark
    P = rs.peers = comm.peers
    _mark(timer, "begin")
    mine = rs.phase_plan(cam)
    _mark(timer, "project_plan")
    comm.counts(mine, rs.cmat)
    rs.phase_sizes()
    _mark(timer, "counts_sync")
    ops = rs.phase_pack()
    _mark(timer, "pack")
    P.barrier() if P is not None else comm.exchange(ops)
    _mark(timer, "exchange_splats")
    to_prev, to_next = rs.phase_render()
    _mark(timer, "bin_render")
    if P is not None:
        P.barrier()
        got_prev = got_next = None
    else:
        sp, sn = rs.halo_shapes()
        got_prev, got_next = comm.halo(to_prev, to_next, sp, sn, torch.float32, rs.dev)
    _mark(timer, "halo")
    parts = rs.phase_loss(got_prev, got_next, gt)
    comm.allreduce_sum_(parts)
    loss = rs.finish_loss()
    _mark(timer, "loss_allreduce")
    gops = rs.phase_backward(timer)
    _mark(timer, "band_fold")
    P.barrier() if P is not None else comm.exchange(gops)
    _mark(timer, "exchange_grads")
    rs.phase_update(it)
    _mark(timer, "owner_fold_chain_adam")
    rs.rebalance()
    return loss


def comm_pair_counts(rs: RankStep, comm: TorchComm, cam) -> dict:
    """Roofline units of this rank's band for view `cam`: pairs
    iterated (I_f), contributing (C) and the backward's I_b (sum of the
    last-contributor index) over the reference's full lists; no state change."""
    P = rs.peers = comm.peers
    comm.counts(rs.phase_plan(cam), rs.cmat)
    rs.phase_sizes()
    ops = rs.phase_pack()
    P.barrier() if P is not None else comm.exchange(ops)
    rs.phase_render(count=True)
    return _band_pair_counts(rs)


def _band_pair_counts(rs: RankStep) -> dict:
    px = (rs.prow1 - rs.prow0) * rs.W
    out = {"M": rs.R, "E": rs.E, "P": px,
           "I_f": int(rs.n_iter[:px].sum(dtype=torch.int64)),
           "C": int(rs.n_contrib[:px].sum(dtype=torch.int64)),
           "I_b": int(rs.n_last[:px].sum(dtype=torch.int64))}
    rs.n_contrib = rs.n_iter = None
    return out


class SpanTimer:
    """Per-rank device time of named phases (CUDA event pairs), for ranks
    whose phases interleave on one stream (the emulated step)."""

    def __init__(self):
        self.spans: list = []

    def span(self, name: str):
        timer = self

        class _Span:
            def __enter__(self_):
                self_.a = torch.cuda.Event(enable_timing=True)
                self_.a.record()

            def __exit__(self_, *exc):
                b = torch.cuda.Event(enable_timing=True)
                b.record()
                timer.spans.append((name, self_.a, b))
                return False
        return _Span()

    def phases(self) -> dict:
        torch.cuda.synchronize()
        out: dict = {}
        for name, a, b in self.spans:
            out[name] = out.get(name, 0.0) + a.elapsed_time(b)
        return out


class _NoSpan:
    def span(self, name):
        import contextlib
        return contextlib.nullcontext()


def _emulated_exchange(ranks: list, ops: list) -> None:
    """Deliver every rank's point-to-point segments by device copies."""
    for src, rank_ops in enumerate(ops):
        for peer, sends, _ in rank_ops:
            recvs = next(r for p, _, r in ops[peer] if p == src)
            for a, b in zip(sends, recvs):
                if a.numel():
                    b.copy_(a)


def emulated_step(ranks: list, cam, gt: torch.Tensor, it: int, timers=None,
                  count: bool = False, peers: bool = False):
    """The same phases for W ranks executed in sequence on ONE GPU with the
    exchanges done by in-process copies (no kernel waits on another rank).
    Used to check bitwise W-invariance on a single B200.  timers: optional
    per-rank SpanTimer list (each rank's device time per phase, i.e. what
    its own GPU would spend outside the exchanges).  count=True: stop after
    the forward with the pair counters (returns the per-rank counts).
    peers=True: the peer-store exchange (EmulatedPeers) -- the pack, halo and
    band-fold kernels store straight into the other ranks' buffers."""
    W = len(ranks)
    tm = timers or [_NoSpan()] * W
    P = EmulatedPeers(ranks) if peers else None
    for r, t in zip(ranks, tm):
        r.peers = P
        with t.span("project_plan"):
            r.phase_plan(cam)
    for dst in range(W):
        for src in range(W):
            ranks[dst].cmat[src].copy_(ranks[src].counts)
    for r in ranks:
        r.phase_sizes()
    ops = []
    for r, t in zip(ranks, tm):
        with t.span("pack"):
            ops.append(r.phase_pack())
    _emulated_exchange(ranks, ops)
    bounds = []
    for r, t in zip(ranks, tm):
        with t.span("bin_render"):
            bounds.append(r.phase_render(count=count))
    if count:
        return [_band_pair_counts(r) for r in ranks]
    for i, (r, t) in enumerate(zip(ranks, tm)):
        got_prev = bounds[i - 1][1] if i > 0 and P is None else None
        got_next = bounds[i + 1][0] if i + 1 < W and P is None else None
        with t.span("loss"):
            r.phase_loss(got_prev, got_next, gt)
    total = torch.zeros_like(ranks[0].parts)
    for r in ranks:
        total += r.parts
    for r in ranks:
        r.parts.copy_(total)
    loss = ranks[0].finish_loss()
    gops = []
    for r, t in zip(ranks, tm):
        with t.span("backward_fold"):
            gops.append(r.phase_backward())
    _emulated_exchange(ranks, gops)
    for r, t in zip(ranks, tm):
        with t.span("owner_fold_chain_adam"):
            r.phase_update(it)
    for r in ranks:
        r.rebalance()
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
    dev = L.require_cuda()
    exchange = getattr(config, "exchange", "peer")
    try:
        comm = TorchComm(peers=exchange == "peer", height=dataset.height, width=dataset.width,
                         device=dev)
    except Exception:  # no symmetric memory / peer mappings: point-to-point copies
        comm = TorchComm(peers=False)
    if comm.world != workers:
        raise ValueError(f"workers={workers} but WORLD_SIZE={comm.world}")
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
