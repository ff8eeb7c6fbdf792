"""Differentiable tile rasteriser: the reference's array API on B200 kernels.

Drop-in for isosplat.rasterizer (/root/reference/pkg/src/isosplat/
rasterizer.py): same names, argument meaning and ValueErrors.  Arrays are CUDA
tensors (numpy inputs are accepted and moved to the device); every compute
step is a libisogs.so kernel -- there is no CPU path.

`dtype` selects the kernel instantiation exactly where the reference has a
`dtype` argument: float32 is the production raster, float64 the tight
cross-check build (bit-identical composite, glibc-exact exp).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .gaussians import GaussianCloud, to_device_cloud

TILE_SIZE = 16


@dataclass(frozen=True)
class ProjectedSplat:
    """rasterizer.py:16-27."""

    gaussian_index: int
    mean2d: np.ndarray
    cov2d: np.ndarray
    depth: float
    color: np.ndarray
    opacity: float
    tile_span: tuple


@dataclass
class SplatBatch:
    """Column-wise projected splats of one view (rasterizer.py:30-69)."""

    indices: torch.Tensor
    mean2d: torch.Tensor
    cov2d: torch.Tensor
    conic: torch.Tensor
    depth: torch.Tensor
    color: torch.Tensor
    opacity: torch.Tensor
    tile_min: torch.Tensor
    tile_max: torch.Tensor
    width: int
    height: int
    tile_size: int
    tiles_x: int
    tiles_y: int

    def __len__(self) -> int:
        return int(self.indices.shape[0])

    def __getitem__(self, i: int) -> ProjectedSplat:
        a, b, c = self.cov2d[i].tolist()
        tmin = self.tile_min[i].tolist()
        tmax = self.tile_max[i].tolist()
        return ProjectedSplat(
            gaussian_index=int(self.indices[i]), mean2d=self.mean2d[i].cpu().numpy(),
            cov2d=np.array([[a, b], [b, c]]), depth=float(self.depth[i]),
            color=self.color[i].cpu().numpy(), opacity=float(self.opacity[i]),
            tile_span=((int(tmin[0]), int(tmin[1])), (int(tmax[0]), int(tmax[1]))))


@dataclass
class RenderAux:
    """rasterizer.py:72-87."""

    t_final: torch.Tensor
    contrib_count: torch.Tensor
    indices: torch.Tensor
    touch_count: torch.Tensor
    grad_norm: torch.Tensor
    width: int
    height: int
    cache: dict = field(default_factory=dict, repr=False)


@dataclass
class ParamGradients:
    """rasterizer.py:90-98."""

    positions: torch.Tensor
    log_scales: torch.Tensor
    rotations: torch.Tensor
    opacity_logits: torch.Tensor
    sh_coeffs: torch.Tensor


# ------------------------------------------------------------------ helpers --

def _dev(x, dtype=None) -> torch.Tensor:
    dev = L.require_cuda()
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(dev).contiguous()


def _params_struct(c: GaussianCloud) -> L.Params_t:
    p = L.Params_t()
    p.positions, p.log_scales, p.rotations = L.ptr(c.positions), L.ptr(c.log_scales), L.ptr(c.rotations)
    p.opacity_logits, p.sh = L.ptr(c.opacity_logits), L.ptr(c.sh_coeffs)
    p.n, p.degree, p.dtype = c.count, int(c.degree), L.dtype_tag(c.dtype)
    return p


def _sortable_f64(x: torch.Tensor) -> torch.Tensor:
    """float64 -> int64 bit keys whose unsigned order is the float order."""
    b = (x.to(torch.float64) + 0.0).view(torch.int64)
    neg = b < 0
    return torch.where(neg, ~b, b | torch.tensor(-(2 ** 63), dtype=torch.int64, device=b.device))


_WS = L.Workspace()
_WS_COMPACT = L.Workspace()


def _stable_argsort_u64(keys: torch.Tensor) -> torch.Tensor:
    vals = torch.arange(keys.numel(), dtype=torch.int32, device=keys.device)
    _, out = L.sort_depth(keys.contiguous(), vals, _WS)
    return out.to(torch.int64)


# -------------------------------------------------------------- projection --

def project(cloud, cam, tile_size: int = TILE_SIZE, indices=None) -> SplatBatch:
    """EWA-project a cloud (or shard) into screen space (rasterizer.py:105-158).

    One isg_preprocess launch (float64, glibc-exact exp) followed by the
    reference's stable compaction of kept rows."""
    if tile_size != TILE_SIZE:
        raise ValueError(f"the B200 kernels use {TILE_SIZE}-px tiles; got {tile_size}")
    dev = L.require_cuda()
    c = cloud if isinstance(cloud, GaussianCloud) and cloud.positions.is_cuda else \
        to_device_cloud(cloud, dev)
    n = c.count
    if indices is None:
        indices = torch.arange(n, dtype=torch.int64, device=dev)
    else:
        indices = _dev(indices, torch.int64)
        if tuple(indices.shape) != (n,):
            raise ValueError(f"indices shape {tuple(indices.shape)} != ({n},)")
    tiles_x = (cam.width + tile_size - 1) // tile_size
    tiles_y = (cam.height + tile_size - 1) // tile_size
    key = torch.empty(n, dtype=torch.int64, device=dev)
    rect = torch.empty((n, 4), dtype=torch.int32, device=dev)
    feat = torch.empty((n, 12), dtype=torch.float32, device=dev)
    flag = torch.empty(n, dtype=torch.uint8, device=dev)
    full = torch.empty((n, 16), dtype=torch.float64, device=dev)
    if n:
        out = L.PreprocessOut_t()
        out.key, out.rect, out.feat = L.ptr(key), L.ptr(rect), L.ptr(feat)
        out.flag, out.full64, out.feat_dtype = L.ptr(flag), L.ptr(full), L.ISG_F32
        p = _params_struct(c)
        cs = L.camera_struct(cam)
        L.check(L.lib().isg_preprocess(ctypes.byref(p), ctypes.byref(cs), tile_size,
                                       ctypes.byref(out), L.stream_ptr()), "isg_preprocess")
    # the stable keep compaction straight into the batch columns
    lib = L.lib()
    pos = torch.empty(n + 1, dtype=torch.int64, device=dev)
    sz = ctypes.c_size_t(0)
    L.check(lib.isg_compact_count(None, ctypes.byref(sz), n, None, None, None), "compact size")
    ws = _WS_COMPACT.get(sz.value, dev)
    sz = ctypes.c_size_t(ws.numel())
    L.check(lib.isg_compact_count(L.ptr(ws), ctypes.byref(sz), n, L.ptr(flag) if n else None,
                                  L.ptr(pos), L.stream_ptr()), "isg_compact_count")
    m = int(pos[n].item())
    f64 = lambda *shape: torch.empty(shape, dtype=torch.float64, device=dev)
    cols = {"mean2d": f64(m, 2), "cov2d": f64(m, 3), "conic": f64(m, 3), "depth": f64(m),
            "color": f64(m, 3), "opacity": f64(m),
            "tile_min": torch.empty((m, 2), dtype=torch.int32, device=dev),
            "tile_max": torch.empty((m, 2), dtype=torch.int32, device=dev),
            "indices": torch.empty(m, dtype=torch.int64, device=dev)}
    if m:
        L.check(lib.isg_compact_batch(n, L.ptr(flag), L.ptr(pos), L.ptr(full), L.ptr(rect),
                                      L.ptr(indices), *(L.ptr(cols[k]) for k in (
                                          "mean2d", "cov2d", "conic", "depth", "color",
                                          "opacity", "tile_min", "tile_max", "indices")),
                                      L.stream_ptr()), "isg_compact_batch")
    return SplatBatch(width=cam.width, height=cam.height, tile_size=tile_size, tiles_x=tiles_x,
                      tiles_y=tiles_y, **cols)


def sort_order(batch: SplatBatch) -> torch.Tensor:
    """np.lexsort((indices, depth)) (rasterizer.py:161-163): two stable radix
    passes -- by global index, then by fp64 depth bits."""
    m = len(batch)
    dev = L.require_cuda()
    if m == 0:
        return torch.empty(0, dtype=torch.int64, device=dev)
    idx = _dev(batch.indices, torch.int64)
    if m > 1 and not bool((idx[1:] >= idx[:-1]).all()):
        perm = _stable_argsort_u64(idx ^ torch.tensor(-(2 ** 63), dtype=torch.int64, device=dev))
    else:
        perm = torch.arange(m, dtype=torch.int64, device=dev)
    depth_keys = _sortable_f64(_dev(batch.depth)[perm])
    return perm[_stable_argsort_u64(depth_keys)]


# ----------------------------------------------------------------- binning --

def _emit_offsets(rect_sorted: torch.Tensor, row_lo: int, row_hi: int) -> torch.Tensor:
    y0 = rect_sorted[:, 1].clamp(min=row_lo)
    y1 = rect_sorted[:, 3].clamp(max=row_hi - 1)
    cnt = ((rect_sorted[:, 2] - rect_sorted[:, 0] + 1).to(torch.int64)
           * (y1 - y0 + 1).clamp(min=0).to(torch.int64))
    off = torch.zeros(rect_sorted.shape[0] + 1, dtype=torch.int64, device=rect_sorted.device)
    torch.cumsum(cnt, 0, out=off[1:])
    return off


def _bin_all_tiles(rect_sorted: torch.Tensor, emit_off: torch.Tensor, tiles_x: int,
                   tiles_y: int) -> tuple[torch.Tensor, torch.Tensor]:
    """CSR over all tiles (offsets int32 (T+1), entries int32 ranks)."""
    dev = rect_sorted.device
    m = rect_sorted.shape[0]
    e = int(emit_off[-1].item()) if m else 0
    n_tiles = tiles_x * tiles_y
    keys = torch.empty(e, dtype=torch.int32, device=dev)
    vals = torch.empty(e, dtype=torch.int32, device=dev)
    if e:
        L.check(L.lib().isg_bin_emit(m, L.ptr(rect_sorted), L.ptr(emit_off), tiles_x, 0, tiles_y,
                                     L.ptr(keys), L.ptr(vals), L.stream_ptr()), "isg_bin_emit")
        bits = max(1, int(n_tiles - 1).bit_length())
        keys, vals = L.sort_pairs(keys, vals, (0, bits), _WS)
    offsets = torch.empty(n_tiles + 1, dtype=torch.int32, device=dev)
    L.check(L.lib().isg_tile_offsets(e, L.ptr(keys) if e else None, n_tiles, L.ptr(offsets),
                                     L.stream_ptr()), "isg_tile_offsets")
    return offsets, vals


def build_tile_lists(sorted_tile_min, sorted_tile_max, own_tiles, tiles_x: int, tiles_y: int):
    """CSR tile lists over ``own_tiles`` (rasterizer.py:166-191).

    Returns (offsets int64 (len(own_tiles)+1), entries int32): entries are
    sorted-splat rows, per tile in compositing order."""
    dev = L.require_cuda()
    rect = torch.cat([_dev(sorted_tile_min, torch.int32), _dev(sorted_tile_max, torch.int32)],
                     1).contiguous()
    own = _dev(own_tiles, torch.int64)
    emit_off = _emit_offsets(rect, 0, tiles_y)
    off_all, ent_all = _bin_all_tiles(rect, emit_off, tiles_x, tiles_y)
    off_all = off_all.to(torch.int64)
    starts = off_all[own]
    counts = off_all[own + 1] - starts
    offsets = torch.zeros(own.numel() + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=offsets[1:])
    total = int(offsets[-1].item())
    if total == 0:
        return offsets, torch.empty(0, dtype=torch.int32, device=dev)
    seg = torch.repeat_interleave(torch.arange(own.numel(), device=dev), counts)
    pos = torch.arange(total, device=dev) - offsets[:-1][seg] + starts[seg]
    return offsets, ent_all[pos].contiguous()


# ------------------------------------------------------------ raster ops ----

def _feat_from(sa: dict, dtype: torch.dtype) -> torch.Tensor:
    m = sa["mean2d"].shape[0]
    dev = sa["mean2d"].device
    return torch.cat([sa["mean2d"].to(dtype), sa["conic"].to(dtype),
                      sa["opacity"].to(dtype).reshape(m, 1), sa["color"].to(dtype),
                      torch.zeros((m, 3), dtype=dtype, device=dev)], 1).contiguous()


def _raster_fwd(feat, offsets32, entries, width, height, tiles_x, tile_ids, bg, image,
                t_final, n_last, n_contrib, touched):
    n_ids = int(tile_ids.numel()) if tile_ids is not None else 0
    rows = (height + TILE_SIZE - 1) // TILE_SIZE
    bgc = (ctypes.c_double * 3)(*[float(v) for v in bg])
    L.check(L.lib().isg_raster_fwd(
        L.dtype_tag(feat.dtype), width, height, tiles_x, 0, rows, L.ptr(tile_ids), n_ids,
        L.ptr(offsets32), L.ptr(entries) if entries.numel() else None, L.ptr(feat) if feat.numel() else None,
        ctypes.cast(bgc, ctypes.c_void_p), L.ptr(image), L.dtype_tag(image.dtype), L.ptr(t_final),
        L.ptr(n_last), L.ptr(n_contrib), None,
        L.ptr(touched) if touched is not None and touched.numel() else None,
        L.stream_ptr()), "isg_raster_fwd")


def forward_on_tiles(sorted_arrays: dict, own_tiles, offsets, entries, width: int, height: int,
                     tiles_x: int, tile_size: int, background, image: torch.Tensor,
                     t_final: torch.Tensor, n_contrib: torch.Tensor, touched: torch.Tensor) -> None:
    """Composite the given tiles into preallocated canvases (rasterizer.py:194-215)."""
    if tile_size != TILE_SIZE:
        raise ValueError(f"the B200 kernels use {TILE_SIZE}-px tiles; got {tile_size}")
    dt = torch.float64 if image.dtype == torch.float64 else torch.float32
    sa = {k: _dev(v) for k, v in sorted_arrays.items() if k in ("mean2d", "conic", "color", "opacity")}
    feat = _feat_from(sa, dt)
    tf = torch.empty(t_final.shape, dtype=dt, device=image.device)
    n_last = torch.empty(t_final.shape, dtype=torch.int32, device=image.device)
    nc = torch.empty(t_final.shape, dtype=torch.int32, device=image.device)
    own = _dev(own_tiles, torch.int32)
    _raster_fwd(feat, _dev(offsets, torch.int32), _dev(entries, torch.int32), width, height,
                tiles_x, own, background, image, tf, n_last, nc, touched)
    # pixels of tiles not listed keep their caller-provided values
    mask = torch.zeros(t_final.shape, dtype=torch.bool, device=image.device)
    tx, ty = own.long() % tiles_x, own.long() // tiles_x
    for k in range(own.numel()):  # small helper loop (API path only)
        y0, x0 = int(ty[k]) * TILE_SIZE, int(tx[k]) * TILE_SIZE
        mask[y0:y0 + TILE_SIZE, x0:x0 + TILE_SIZE] = True
    t_final[mask] = tf[mask].to(t_final.dtype)
    n_contrib[mask] = nc[mask]


def backward_on_tiles(sorted_arrays: dict, own_tiles, offsets, entries, width: int, height: int,
                      tiles_x: int, tile_size: int, background, dl_dimage) -> dict:
    """Per-(tile, splat) gradient subtotals, rows aligned with entries
    (rasterizer.py:218-245).  Runs the float64 instantiation like the
    reference's scratch (float64)."""
    if tile_size != TILE_SIZE:
        raise ValueError(f"the B200 kernels use {TILE_SIZE}-px tiles; got {tile_size}")
    sa = {k: _dev(v) for k, v in sorted_arrays.items() if k in ("mean2d", "conic", "color", "opacity")}
    feat = _feat_from(sa, torch.float64)
    dev = feat.device
    own = _dev(own_tiles, torch.int32)
    off32 = _dev(offsets, torch.int32)
    ent = _dev(entries, torch.int32)
    e = int(ent.numel())
    # forward replay to obtain T_final / last contributor per pixel
    image = torch.empty((height, width, 3), dtype=torch.float64, device=dev)
    tf = torch.ones((height, width), dtype=torch.float64, device=dev)
    n_last = torch.zeros((height, width), dtype=torch.int32, device=dev)
    _raster_fwd(feat, off32, ent, width, height, tiles_x, own, background, image, tf, n_last,
                None, None)
    partials = torch.zeros((max(e, 1), 9), dtype=torch.float64, device=dev)
    dl = _dev(dl_dimage)
    bgc = (ctypes.c_double * 3)(*[float(v) for v in background])
    rows = (height + TILE_SIZE - 1) // TILE_SIZE
    L.check(L.lib().isg_raster_bwd(
        L.ISG_F64, width, height, tiles_x, 0, rows, L.ptr(own), int(own.numel()), L.ptr(off32),
        L.ptr(ent) if e else None, L.ptr(feat) if feat.numel() else None, None, None,
        ctypes.cast(bgc, ctypes.c_void_p), L.ptr(tf), L.ptr(n_last), L.ptr(dl),
        L.dtype_tag(dl.dtype), L.ptr(partials), L.stream_ptr()), "isg_raster_bwd")
    partials = partials[:e]
    return {"dmean": partials[:, 0:2].contiguous(), "dconic": partials[:, 2:5].contiguous(),
            "dcolor": partials[:, 5:8].contiguous(), "dopac": partials[:, 8].contiguous()}


def reduce_scratch(entries, scratch: dict, m: int) -> dict:
    """Fold per-(tile, splat) subtotals in entry (ascending tile) order
    (_kernels.py:398-411) with isg_reduce_ordered."""
    dev = L.require_cuda()
    ent = _dev(entries, torch.int64)
    part = torch.cat([_dev(scratch["dmean"]), _dev(scratch["dconic"]), _dev(scratch["dcolor"]),
                      _dev(scratch["dopac"]).reshape(-1, 1)], 1).to(torch.float64)
    perm = _stable_argsort_u64(ent)  # splat-major, tile order kept (stable)
    part = part[perm].contiguous()
    counts = torch.bincount(ent, minlength=m)[:m]
    off = torch.zeros(m + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=off[1:])
    g2d = torch.zeros((m, 9), dtype=torch.float64, device=dev)
    order = torch.arange(m, dtype=torch.int32, device=dev)
    if m:
        L.check(L.lib().isg_reduce_ordered(L.ISG_F64, m, L.ptr(off), L.ptr(part) if part.numel() else None,
                                           L.ptr(order), None, 0, 0, 0, L.ptr(g2d), None,
                                           L.stream_ptr()), "isg_reduce_ordered")
    return {"dmean": g2d[:, 0:2], "dconic": g2d[:, 2:5], "dcolor": g2d[:, 5:8], "dopac": g2d[:, 8]}


def chain_to_params(cloud, cam, flags, acc_dmean, acc_dconic, acc_dcolor, acc_dopac) -> ParamGradients:
    """2D splat gradients -> 3D parameter gradients (rasterizer.py:248-280)."""
    dev = L.require_cuda()
    c = cloud if isinstance(cloud, GaussianCloud) and cloud.positions.is_cuda else \
        to_device_cloud(cloud, dev)
    n = c.count
    g2d = torch.cat([_dev(acc_dmean, torch.float64).reshape(n, 2),
                     _dev(acc_dconic, torch.float64).reshape(n, 3),
                     _dev(acc_dcolor, torch.float64).reshape(n, 3),
                     _dev(acc_dopac, torch.float64).reshape(n, 1)], 1).contiguous()
    return _chain(c, cam, _dev(flags, torch.uint8), g2d)


def _chain(c: GaussianCloud, cam, flags: torch.Tensor, g2d: torch.Tensor) -> ParamGradients:
    out = ParamGradients(*(torch.empty_like(getattr(c, k)) for k in
                           ("positions", "log_scales", "rotations", "opacity_logits", "sh_coeffs")))
    if c.count:
        p = _params_struct(c)
        cs = L.camera_struct(cam)
        L.check(L.lib().isg_chain(ctypes.byref(p), ctypes.byref(cs), L.ptr(flags), L.ptr(g2d),
                                  L.ptr(out.positions), L.ptr(out.log_scales),
                                  L.ptr(out.rotations), L.ptr(out.opacity_logits),
                                  L.ptr(out.sh_coeffs), L.stream_ptr()), "isg_chain")
    return out


# --------------------------------------------------------- render (public) --

def render_forward(batch: SplatBatch, width: int, height: int,
                   background=(1.0, 1.0, 1.0), tile_size: int = TILE_SIZE,
                   dtype=torch.float32):
    """Composite a projected batch front-to-back (rasterizer.py:294-345).

    Returns (image (H,W,3) of `dtype`, RenderAux, order)."""
    if width != batch.width or height != batch.height or tile_size != batch.tile_size:
        raise ValueError("render dims must match the projecting camera")
    if tile_size != TILE_SIZE:
        raise ValueError(f"the B200 kernels use {TILE_SIZE}-px tiles; got {tile_size}")
    dt = _torch_dtype(dtype)
    dev = L.require_cuda()
    m = len(batch)
    order = sort_order(batch)
    rect = torch.empty((m, 4), dtype=torch.int32, device=dev)
    feat = torch.empty((m, 12), dtype=dt, device=dev)
    if m:
        cols = [_dev(getattr(batch, k), torch.float64) for k in ("mean2d", "conic", "color",
                                                                 "opacity")]
        tmin, tmax = _dev(batch.tile_min, torch.int32), _dev(batch.tile_max, torch.int32)
        L.check(L.lib().isg_gather_batch(m, L.ptr(order), *(L.ptr(c) for c in cols),
                                         L.ptr(tmin), L.ptr(tmax), L.dtype_tag(dt), L.ptr(feat),
                                         L.ptr(rect), L.stream_ptr()), "isg_gather_batch")
    emit_off = _emit_offsets(rect, 0, batch.tiles_y)
    offsets, entries = _bin_all_tiles(rect, emit_off, batch.tiles_x, batch.tiles_y)
    image = torch.empty((height, width, 3), dtype=dt, device=dev)
    t_final = torch.empty((height, width), dtype=dt, device=dev)
    n_last = torch.empty((height, width), dtype=torch.int32, device=dev)
    n_contrib = torch.empty((height, width), dtype=torch.int32, device=dev)
    touched_sorted = torch.zeros(m, dtype=torch.int64, device=dev)
    _raster_fwd(feat, offsets, entries, width, height, batch.tiles_x, None, background, image,
                t_final, n_last, n_contrib, touched_sorted)
    touched = torch.zeros(m, dtype=torch.int64, device=dev)
    touched[order] = touched_sorted
    aux = RenderAux(
        t_final=t_final.to(torch.float64), contrib_count=n_contrib,
        indices=batch.indices.clone(), touch_count=touched,
        grad_norm=torch.zeros(m, dtype=torch.float64, device=dev), width=width, height=height,
        cache={"feat": feat, "rect": rect, "emit_off": emit_off, "offsets": offsets,
               "entries": entries, "order": order, "t_final": t_final, "n_last": n_last,
               "background": tuple(float(v) for v in background), "tiles_x": batch.tiles_x,
               "tiles_y": batch.tiles_y, "tile_size": tile_size})
    return image, aux, order


def render_backward(cloud, cam, batch: SplatBatch, order, aux: RenderAux,
                    dl_dimage) -> ParamGradients:
    """Analytic gradients of the forward render (rasterizer.py:348-411)."""
    cache = aux.cache
    if not cache or cache.get("order") is None:
        raise ValueError("aux does not carry forward-pass context")
    order = _dev(order, torch.int64)
    if order.shape != cache["order"].shape or not torch.equal(order, cache["order"]):
        raise ValueError("sort order does not match the forward pass")
    dl = _dev(dl_dimage)
    if tuple(dl.shape) != (aux.height, aux.width, 3):
        raise ValueError(f"dL/dImage shape {tuple(dl.shape)} != {(aux.height, aux.width, 3)}")
    if len(batch) != order.shape[0] or not torch.equal(_dev(aux.indices), _dev(batch.indices)):
        raise ValueError("batch does not match the forward pass")
    dev = dl.device
    m = len(batch)
    feat = cache["feat"]
    e = int(cache["entries"].numel())
    rec = 12 if feat.dtype == torch.float32 else 9  # padded float32 records (isogs.h)
    partials = torch.empty((max(e, 1), rec), dtype=feat.dtype, device=dev)
    bgc = (ctypes.c_double * 3)(*cache["background"])
    if m:
        L.check(L.lib().isg_raster_bwd(
            L.dtype_tag(feat.dtype), aux.width, aux.height, cache["tiles_x"], 0, cache["tiles_y"],
            None, 0, L.ptr(cache["offsets"]), L.ptr(cache["entries"]) if e else None, L.ptr(feat),
            L.ptr(cache["rect"]), L.ptr(cache["emit_off"]), ctypes.cast(bgc, ctypes.c_void_p),
            L.ptr(cache["t_final"]), L.ptr(cache["n_last"]), L.ptr(dl), L.dtype_tag(dl.dtype),
            L.ptr(partials), L.stream_ptr()), "isg_raster_bwd")
    g2d_b = torch.zeros((m, 9), dtype=torch.float64, device=dev)
    gnorm = torch.zeros(m, dtype=torch.float64, device=dev)
    if m:
        L.check(L.lib().isg_reduce_ordered(
            L.dtype_tag(feat.dtype), m, L.ptr(cache["emit_off"]), L.ptr(partials),
            L.ptr(order.to(torch.int32)), None, 0, 0, 0, L.ptr(g2d_b), L.ptr(gnorm),
            L.stream_ptr()),
            "isg_reduce_ordered")
    aux.grad_norm.copy_(gnorm)
    c = cloud if isinstance(cloud, GaussianCloud) and cloud.positions.is_cuda else \
        to_device_cloud(cloud, dev)
    n = c.count
    rows = _dev(batch.indices, torch.int64)
    flags = torch.zeros(n, dtype=torch.uint8, device=dev)
    flags[rows] = 1
    full = torch.zeros((n, 9), dtype=torch.float64, device=dev)
    full[rows] = g2d_b
    return _chain(c, cam, flags, full)


def _torch_dtype(dtype) -> torch.dtype:
    if dtype in (torch.float32, np.float32) or dtype == np.dtype(np.float32):
        return torch.float32
    if dtype in (torch.float64, np.float64) or dtype == np.dtype(np.float64):
        return torch.float64
    raise ValueError(f"unsupported dtype {dtype}")
