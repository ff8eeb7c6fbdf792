"""CPU oracle for the training-step hot path -- TEST INFRASTRUCTURE ONLY.

Python face of ``oracle/isg_oracle.c`` with the reference's array API
(``isosplat`` 0.1.0, paths relative to /root/reference/pkg/src/isosplat/).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module; the product package never does.

Arrays are numpy; every function follows the reference function cited in its
docstring, with the numba kernels replaced by the C restatement and the numpy
glue (lexsort, cumsum, scatter) kept as the reference writes it.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liborc.so")
_lib = None

TILE_SIZE = 16
ADAM_BETA1 = 0.9
ADAM_BETA2 = 0.999
ADAM_EPS = 1e-15


def build() -> str:
    """Compile the C restatement (gcc, -ffp-contract=off) into oracle/_build."""
    src = os.path.join(_HERE, "isg_oracle.c")
    if (not os.path.exists(_LIB_PATH)
            or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src)):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


class _Cam(ctypes.Structure):
    _fields_ = [("R", ctypes.c_double * 9), ("t", ctypes.c_double * 3),
                ("C", ctypes.c_double * 3), ("fx", ctypes.c_double),
                ("fy", ctypes.c_double), ("cx", ctypes.c_double),
                ("cy", ctypes.c_double), ("width", ctypes.c_int32),
                ("height", ctypes.c_int32)]


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.orc_loss_l1_dssim.restype = ctypes.c_double
        _lib.orc_ssim.restype = ctypes.c_double
        _lib.orc_num_threads.restype = ctypes.c_int
    return _lib


def num_threads() -> int:
    return int(lib().orc_num_threads())


class _Ptr(ctypes.c_void_p):
    """void* that keeps the numpy array it points into alive for the call."""


def _p(a: np.ndarray):
    ptr = _Ptr(a.ctypes.data if a.size else 0)
    ptr._keep = a
    return ptr


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _cam_struct(cam) -> _Cam:
    c = _Cam()
    r = np.asarray(cam.rotation, dtype=np.float64).reshape(9)
    t = np.asarray(cam.translation, dtype=np.float64).reshape(3)
    pos = -np.asarray(cam.rotation, dtype=np.float64).T @ t
    for i in range(9):
        c.R[i] = float(r[i])
    for i in range(3):
        c.t[i] = float(t[i])
        c.C[i] = float(pos[i])
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.width, c.height = int(cam.width), int(cam.height)
    return c


@dataclass
class SplatBatch:
    """rasterizer.py:30-56."""

    indices: np.ndarray
    mean2d: np.ndarray
    cov2d: np.ndarray
    conic: np.ndarray
    depth: np.ndarray
    color: np.ndarray
    opacity: np.ndarray
    tile_min: np.ndarray
    tile_max: np.ndarray
    width: int
    height: int
    tile_size: int
    tiles_x: int
    tiles_y: int

    def __len__(self) -> int:
        return self.indices.shape[0]


@dataclass
class RenderAux:
    """rasterizer.py:72-87."""

    t_final: np.ndarray
    contrib_count: np.ndarray
    indices: np.ndarray
    touch_count: np.ndarray
    grad_norm: np.ndarray
    width: int
    height: int
    cache: dict = field(default_factory=dict, repr=False)


@dataclass
class ParamGradients:
    """rasterizer.py:90-98."""

    positions: np.ndarray
    log_scales: np.ndarray
    rotations: np.ndarray
    opacity_logits: np.ndarray
    sh_coeffs: np.ndarray


def project(cloud, cam, tile_size: int = TILE_SIZE, indices=None) -> SplatBatch:
    """rasterizer.py:105-158 over _kernels.py:144-198."""
    n = cloud.positions.shape[0]
    if indices is None:
        indices = np.arange(n, dtype=np.int64)
    else:
        indices = np.asarray(indices, dtype=np.int64)
        if indices.shape != (n,):
            raise ValueError(f"indices shape {indices.shape} != ({n},)")
    tiles_x = (cam.width + tile_size - 1) // tile_size
    tiles_y = (cam.height + tile_size - 1) // tile_size
    flag = np.zeros(n, dtype=np.uint8)
    mean2d = np.empty((n, 2))
    cov2d = np.empty((n, 3))
    conic = np.empty((n, 3))
    depth = np.empty(n)
    color = np.empty((n, 3))
    opacity = np.empty(n)
    tiles = np.empty((n, 4), dtype=np.int32)
    if n:
        pos, ls, rot = _f64(cloud.positions), _f64(cloud.log_scales), _f64(cloud.rotations)
        lg, sh = _f64(cloud.opacity_logits), _f64(cloud.sh_coeffs)
        c = _cam_struct(cam)
        lib().orc_project(
            ctypes.c_int64(n), _p(pos), _p(ls), _p(rot), _p(lg), _p(sh),
            ctypes.c_int(int(cloud.degree)), ctypes.byref(c), ctypes.c_int(tile_size),
            ctypes.c_int(tiles_x), ctypes.c_int(tiles_y), _p(flag), _p(mean2d),
            _p(cov2d), _p(conic), _p(depth), _p(color), _p(opacity), _p(tiles))
    keep = flag.astype(bool)
    return SplatBatch(
        indices=indices[keep], mean2d=mean2d[keep], cov2d=cov2d[keep],
        conic=conic[keep], depth=depth[keep], color=color[keep],
        opacity=opacity[keep], tile_min=tiles[keep][:, 0:2].copy(),
        tile_max=tiles[keep][:, 2:4].copy(), width=cam.width, height=cam.height,
        tile_size=tile_size, tiles_x=tiles_x, tiles_y=tiles_y)


def sort_order(batch: SplatBatch) -> np.ndarray:
    """rasterizer.py:161-163."""
    return np.lexsort((batch.indices, batch.depth))


def build_tile_lists(sorted_tile_min, sorted_tile_max, own_tiles, tiles_x, tiles_y):
    """rasterizer.py:166-191 over _kernels.py:202-225."""
    n_tiles = tiles_x * tiles_y
    own_tiles = np.ascontiguousarray(own_tiles, dtype=np.int32)
    tile_slot = np.full(n_tiles, -1, dtype=np.int32)
    tile_slot[own_tiles] = np.arange(own_tiles.shape[0], dtype=np.int32)
    rects = np.ascontiguousarray(
        np.concatenate([sorted_tile_min, sorted_tile_max], axis=1).astype(np.int32))
    m = rects.shape[0]
    counts = np.zeros(own_tiles.shape[0], dtype=np.int64)
    if m:
        lib().orc_count_tile_entries(ctypes.c_int64(m), _p(rects), _p(tile_slot),
                                     ctypes.c_int(tiles_x), _p(counts))
    offsets = np.zeros(own_tiles.shape[0] + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    entries = np.empty(offsets[-1], dtype=np.int32)
    cursor = np.zeros(own_tiles.shape[0], dtype=np.int64)
    if m:
        lib().orc_fill_tile_entries(ctypes.c_int64(m), _p(rects), _p(tile_slot),
                                    ctypes.c_int(tiles_x), _p(offsets), _p(cursor),
                                    _p(entries))
    return offsets, entries


def _sorted_arrays(batch: SplatBatch, order: np.ndarray) -> dict:
    """rasterizer.py:283-291."""
    return {
        "mean2d": _f64(batch.mean2d[order]), "conic": _f64(batch.conic[order]),
        "color": _f64(batch.color[order]), "opacity": _f64(batch.opacity[order]),
        "tile_min": batch.tile_min[order], "tile_max": batch.tile_max[order],
    }


def forward_on_tiles(sa, own_tiles, offsets, entries, width, height, tiles_x,
                     tile_size, background, image, t_final, n_contrib, touched):
    """rasterizer.py:194-215 over _kernels.py:229-278.  ``image`` may be f32 or
    f64; the composite runs in f64 and is stored with a single rounding."""
    own_tiles = np.ascontiguousarray(own_tiles, dtype=np.int32)
    img64 = np.ascontiguousarray(image, dtype=np.float64)
    tf = np.ascontiguousarray(t_final, dtype=np.float64)
    nc = np.ascontiguousarray(n_contrib, dtype=np.int32)
    bg = _f64(background)
    touched_buf = np.ascontiguousarray(touched, dtype=np.int64)
    lib().orc_forward_tiles(
        ctypes.c_int64(own_tiles.shape[0]), _p(own_tiles), _p(np.ascontiguousarray(offsets, dtype=np.int64)),
        _p(np.ascontiguousarray(entries, dtype=np.int32)), _p(sa["mean2d"]), _p(sa["conic"]),
        _p(sa["color"]), _p(sa["opacity"]), ctypes.c_int(tiles_x), ctypes.c_int(tile_size),
        ctypes.c_int(width), ctypes.c_int(height), _p(bg), _p(img64), _p(tf), _p(nc),
        _p(touched_buf) if touched_buf.size else ctypes.c_void_p(0))
    image[...] = img64
    t_final[...] = tf
    n_contrib[...] = nc
    touched[...] = touched_buf


def backward_on_tiles(sa, own_tiles, offsets, entries, width, height, tiles_x,
                      tile_size, background, dl_dimage) -> dict:
    """rasterizer.py:218-245 over _kernels.py:282-374."""
    e = entries.shape[0]
    scratch = {"dmean": np.zeros((e, 2)), "dconic": np.zeros((e, 3)),
               "dcolor": np.zeros((e, 3)), "dopac": np.zeros(e)}
    own_tiles = np.ascontiguousarray(own_tiles, dtype=np.int32)
    dl = _f64(dl_dimage)
    lib().orc_backward_tiles(
        ctypes.c_int64(own_tiles.shape[0]), _p(own_tiles), _p(np.ascontiguousarray(offsets, dtype=np.int64)),
        _p(np.ascontiguousarray(entries, dtype=np.int32)), _p(sa["mean2d"]), _p(sa["conic"]),
        _p(sa["color"]), _p(sa["opacity"]), ctypes.c_int(tiles_x), ctypes.c_int(tile_size),
        ctypes.c_int(width), ctypes.c_int(height), _p(_f64(background)), _p(dl),
        _p(scratch["dmean"]), _p(scratch["dconic"]), _p(scratch["dcolor"]), _p(scratch["dopac"]))
    return scratch


def reduce_scratch(entries, scratch, m):
    """_kernels.py:398-411: fold per-(tile, splat) subtotals in entry order."""
    acc = {"dmean": np.zeros((m, 2)), "dconic": np.zeros((m, 3)),
           "dcolor": np.zeros((m, 3)), "dopac": np.zeros(m)}
    if m and entries.shape[0]:
        lib().orc_reduce_scratch(
            ctypes.c_int64(entries.shape[0]), _p(np.ascontiguousarray(entries, dtype=np.int32)),
            _p(scratch["dmean"]), _p(scratch["dconic"]), _p(scratch["dcolor"]),
            _p(scratch["dopac"]), _p(acc["dmean"]), _p(acc["dconic"]),
            _p(acc["dcolor"]), _p(acc["dopac"]))
    return acc


def chain_to_params(cloud, cam, flags, acc_dmean, acc_dconic, acc_dcolor, acc_dopac):
    """rasterizer.py:248-280 over _kernels.py:415-634."""
    n = cloud.positions.shape[0]
    k = (cloud.degree + 1) ** 2
    dpos = np.zeros((n, 3))
    dls = np.zeros((n, 3))
    drot = np.zeros((n, 4))
    dlogit = np.zeros(n)
    dsh = np.zeros((n, k, 3))
    if n:
        c = _cam_struct(cam)
        lib().orc_chain(
            ctypes.c_int64(n), _p(_f64(cloud.positions)), _p(_f64(cloud.log_scales)),
            _p(_f64(cloud.rotations)), _p(_f64(cloud.opacity_logits)), _p(_f64(cloud.sh_coeffs)),
            ctypes.c_int(int(cloud.degree)), ctypes.byref(c),
            _p(np.ascontiguousarray(flags, dtype=np.uint8)), _p(_f64(acc_dmean)),
            _p(_f64(acc_dconic)), _p(_f64(acc_dcolor)), _p(_f64(acc_dopac)),
            _p(dpos), _p(dls), _p(drot), _p(dlogit), _p(dsh))
    dt = np.asarray(cloud.positions).dtype
    return ParamGradients(positions=dpos.astype(dt), log_scales=dls.astype(dt),
                          rotations=drot.astype(dt), opacity_logits=dlogit.astype(dt),
                          sh_coeffs=dsh.astype(dt))


def render_forward(batch: SplatBatch, width, height, background=(1.0, 1.0, 1.0),
                   tile_size: int = TILE_SIZE, dtype=np.float32):
    """rasterizer.py:294-345."""
    if width != batch.width or height != batch.height or tile_size != batch.tile_size:
        raise ValueError("render dims must match the projecting camera")
    order = sort_order(batch)
    sa = _sorted_arrays(batch, order)
    own_tiles = np.arange(batch.tiles_x * batch.tiles_y, dtype=np.int32)
    offsets, entries = build_tile_lists(sa["tile_min"], sa["tile_max"], own_tiles,
                                        batch.tiles_x, batch.tiles_y)
    image = np.zeros((height, width, 3), dtype=dtype)
    t_final = np.ones((height, width), dtype=np.float64)
    n_contrib = np.zeros((height, width), dtype=np.int32)
    touched_sorted = np.zeros(len(batch), dtype=np.int64)
    bg = np.asarray(background, dtype=np.float64)
    forward_on_tiles(sa, own_tiles, offsets, entries, width, height, batch.tiles_x,
                     tile_size, bg, image, t_final, n_contrib, touched_sorted)
    touched = np.zeros(len(batch), dtype=np.int64)
    touched[order] = touched_sorted
    aux = RenderAux(t_final=t_final, contrib_count=n_contrib, indices=batch.indices.copy(),
                    touch_count=touched, grad_norm=np.zeros(len(batch)), width=width,
                    height=height,
                    cache={"sorted": sa, "own_tiles": own_tiles, "offsets": offsets,
                           "entries": entries, "order": order, "background": bg,
                           "tiles_x": batch.tiles_x, "tile_size": tile_size})
    return image, aux, order


def render_backward_2d(batch: SplatBatch, order, aux: RenderAux, dl_dimage):
    """rasterizer.py:374-397: per-splat 2D gradients in batch-row order."""
    cache = aux.cache
    m = len(batch)
    scratch = backward_on_tiles(cache["sorted"], cache["own_tiles"], cache["offsets"],
                                cache["entries"], aux.width, aux.height, cache["tiles_x"],
                                cache["tile_size"], cache["background"], dl_dimage)
    acc = reduce_scratch(cache["entries"], scratch, m)
    out = {}
    for key in ("dmean", "dconic", "dcolor", "dopac"):
        b = np.zeros_like(acc[key])
        b[order] = acc[key]
        out[key] = b
    aux.grad_norm[:] = np.hypot(out["dmean"][:, 0], out["dmean"][:, 1])
    return out, scratch


def render_backward(cloud, cam, batch: SplatBatch, order, aux: RenderAux, dl_dimage):
    """rasterizer.py:348-411."""
    cache = aux.cache
    if not cache or cache.get("order") is None:
        raise ValueError("aux does not carry forward-pass context")
    if order.shape != cache["order"].shape or not np.array_equal(order, cache["order"]):
        raise ValueError("sort order does not match the forward pass")
    if dl_dimage.shape != (aux.height, aux.width, 3):
        raise ValueError("dL/dImage shape mismatch")
    b2d, _ = render_backward_2d(batch, order, aux, dl_dimage)
    n = cloud.positions.shape[0]
    flags = np.zeros(n, dtype=np.uint8)
    full = {k: np.zeros((n,) + v.shape[1:]) for k, v in b2d.items()}
    rows = batch.indices
    flags[rows] = 1
    for k in full:
        full[k][rows] = b2d[k]
    return chain_to_params(cloud, cam, flags, full["dmean"], full["dconic"],
                           full["dcolor"], full["dopac"])


def loss_l1_dssim(img, ref, lambda_dssim: float = 0.2):
    """metrics.py:135-189."""
    if not 0.0 <= lambda_dssim <= 1.0:
        raise ValueError("lambda_dssim must lie in [0, 1]")
    a = _f64(img)
    b = _f64(ref)
    if a.shape != b.shape or a.ndim != 3 or a.shape[2] != 3:
        raise ValueError("expected matching (H, W, 3) images")
    h, w = a.shape[:2]
    if h < 11 or w < 11:
        raise ValueError("image smaller than the SSIM window")
    grad = np.empty_like(a)
    loss = lib().orc_loss_l1_dssim(ctypes.c_int(h), ctypes.c_int(w), _p(a), _p(b),
                                   ctypes.c_double(float(lambda_dssim)), _p(grad))
    out_dtype = np.asarray(img).dtype
    if grad.dtype != out_dtype:
        grad = grad.astype(out_dtype)
    return float(loss), grad


def ssim(img, ref) -> float:
    """metrics.py:105-132."""
    a = _f64(img)
    b = _f64(ref)
    if a.ndim == 2:
        a = a[:, :, None].copy()
        b = b[:, :, None].copy()
    h, w, c = a.shape
    return float(lib().orc_ssim(ctypes.c_int(h), ctypes.c_int(w), ctypes.c_int(c),
                                _p(a), _p(b)))


def psnr(img, ref) -> float:
    """metrics.py:75-84."""
    a = np.asarray(img, dtype=np.float64)
    b = np.asarray(ref, dtype=np.float64)
    mse = float(np.mean((a - b) ** 2))
    if mse == 0.0:
        return 100.0
    return min(-10.0 * math.log10(mse), 100.0)


def quantize8(img):
    """images.py:9-16."""
    q = np.rint(np.clip(np.asarray(img, dtype=np.float64), 0.0, 1.0) * 255.0)
    return q / 255.0


def adam_step(params: dict, grads: dict, state: dict, iteration: int, lrs: dict,
              beta1=ADAM_BETA1, beta2=ADAM_BETA2, eps=ADAM_EPS):
    """optim.py:20-56 (numpy weak-scalar semantics: constants rounded to the
    array dtype before each elementwise op)."""
    if iteration < 1:
        raise ValueError("iteration must be >= 1")
    bc1 = 1.0 - beta1 ** iteration
    bc2 = 1.0 - beta2 ** iteration
    for name, p in params.items():
        g = np.ascontiguousarray(grads[name], dtype=p.dtype)
        st = state[name]
        m, v = st["m"], st["v"]
        if p.dtype == np.float32:
            f = np.float32
            lib().orc_adam_f32(ctypes.c_int64(p.size), _p(p), _p(g), _p(m), _p(v),
                               ctypes.c_float(f(beta1)), ctypes.c_float(f(1.0 - beta1)),
                               ctypes.c_float(f(beta2)), ctypes.c_float(f(1.0 - beta2)),
                               ctypes.c_float(f(bc1)), ctypes.c_float(f(bc2)),
                               ctypes.c_float(f(lrs[name])), ctypes.c_float(f(eps)))
        else:
            lib().orc_adam_f64(ctypes.c_int64(p.size), _p(p), _p(g), _p(m), _p(v),
                               ctypes.c_double(beta1), ctypes.c_double(1.0 - beta1),
                               ctypes.c_double(beta2), ctypes.c_double(1.0 - beta2),
                               ctypes.c_double(bc1), ctypes.c_double(bc2),
                               ctypes.c_double(lrs[name]), ctypes.c_double(eps))
    return params, state


def route_mask(tile_min, tile_max, workers, tiles_x):
    """distributed.py:127-136 over _kernels.py:378-394."""
    n = tile_min.shape[0]
    mask = np.zeros((n, workers), dtype=np.uint8)
    if n:
        rects = np.ascontiguousarray(np.concatenate([tile_min, tile_max], axis=1).astype(np.int32))
        lib().orc_route_mask(ctypes.c_int64(n), _p(rects), ctypes.c_int(tiles_x),
                             ctypes.c_int(workers), _p(mask))
    return mask
