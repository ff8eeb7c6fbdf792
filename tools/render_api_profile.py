"""Where the public render_forward's time goes (CUDA events around each of
its steps, config from argv)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2509_05216_b200 as P
from paper_2509_05216_b200 import rasterizer as R
from paper_2509_05216_b200 import synthetic as S

name = sys.argv[1] if len(sys.argv) > 1 else "config3"
dev = torch.device("cuda", 0)
wl = S.make_workload(name, dev, view_ids=[0, 1])
cloud = P.cloud_from_points(wl.points, wl.log_scales, 1, dev)
cam = wl.cameras[0]
res = wl.resolution
for rep in range(3):
    ev = []
    def mark(tag):
        e = torch.cuda.Event(enable_timing=True); e.record(); ev.append((tag, e))
    torch.cuda.synchronize(); mark("start")
    batch = P.project(cloud, cam); mark("project")
    order = R.sort_order(batch); mark("sort_order")
    m = len(batch)
    rect = torch.empty((m, 4), dtype=torch.int32, device=dev)
    feat = torch.empty((m, 12), dtype=torch.float32, device=dev)
    R.L.check(R.L.lib().isg_gather_batch(m, R.L.ptr(order), R.L.ptr(batch.mean2d),
                                         R.L.ptr(batch.conic), R.L.ptr(batch.color),
                                         R.L.ptr(batch.opacity), R.L.ptr(batch.tile_min),
                                         R.L.ptr(batch.tile_max), R.L.ISG_F32, R.L.ptr(feat),
                                         R.L.ptr(rect), R.L.stream_ptr()), "gather")
    mark("gather+feat")
    emit_off = R._emit_offsets(rect, 0, batch.tiles_y); mark("emit_offsets")
    offsets, entries = R._bin_all_tiles(rect, emit_off, batch.tiles_x, batch.tiles_y); mark("bin_all_tiles")
    m = len(batch)
    image = torch.empty((res, res, 3), dtype=torch.float32, device=dev)
    t_final = torch.empty((res, res), dtype=torch.float32, device=dev)
    n_last = torch.empty((res, res), dtype=torch.int32, device=dev)
    n_contrib = torch.empty((res, res), dtype=torch.int32, device=dev)
    touched_sorted = torch.zeros(m, dtype=torch.int64, device=dev)
    R._raster_fwd(feat, offsets, entries, res, res, batch.tiles_x, None, (1.0, 1.0, 1.0), image,
                  t_final, n_last, n_contrib, touched_sorted); mark("raster_fwd")
    touched = torch.zeros(m, dtype=torch.int64, device=dev); touched[order] = touched_sorted
    t64 = t_final.to(torch.float64); idx = batch.indices.clone(); mark("aux")
    torch.cuda.synchronize()
    print({tag: round(ev[i - 1][1].elapsed_time(e), 3) for i, (tag, e) in enumerate(ev) if i},
          "m", m, "e", int(entries.numel()))

# render_backward's steps
img, aux, order = P.render_forward(P.project(cloud, cam), res, res)
batch = P.project(cloud, cam)
dl = torch.full((res, res, 3), 1e-3, dtype=torch.float32, device=dev)
import ctypes
for rep in range(2):
    ev = []
    def mark(tag):
        e = torch.cuda.Event(enable_timing=True); e.record(); ev.append((tag, e))
    torch.cuda.synchronize(); mark("start")
    cache = aux.cache
    o = R._dev(order, torch.int64)
    ok = o.shape == cache["order"].shape and torch.equal(o, cache["order"])
    ok2 = torch.equal(R._dev(aux.indices), R._dev(batch.indices)); mark("checks")
    feat = cache["feat"]; e_ = int(cache["entries"].numel()); m = len(batch)
    partials = torch.empty((max(e_, 1), 12), dtype=feat.dtype, device=dev)
    bgc = (ctypes.c_double * 3)(*cache["background"])
    R.L.check(R.L.lib().isg_raster_bwd(R.L.dtype_tag(feat.dtype), aux.width, aux.height, cache["tiles_x"], 0, cache["tiles_y"], None, 0, R.L.ptr(cache["offsets"]), R.L.ptr(cache["entries"]), R.L.ptr(feat), R.L.ptr(cache["rect"]), R.L.ptr(cache["emit_off"]), ctypes.cast(bgc, ctypes.c_void_p), R.L.ptr(cache["t_final"]), R.L.ptr(cache["n_last"]), R.L.ptr(dl), R.L.dtype_tag(dl.dtype), R.L.ptr(partials), R.L.stream_ptr()), "bwd"); mark("raster_bwd")
    g2d = torch.zeros((m, 9), dtype=torch.float64, device=dev); gn = torch.zeros(m, dtype=torch.float64, device=dev)
    R.L.check(R.L.lib().isg_reduce_ordered(R.L.dtype_tag(feat.dtype), m, R.L.ptr(cache["emit_off"]), R.L.ptr(partials), R.L.ptr(o.to(torch.int32)), None, 0, 0, 0, R.L.ptr(g2d), R.L.ptr(gn), R.L.stream_ptr()), "reduce"); mark("reduce")
    n = cloud.count
    rows = R._dev(batch.indices, torch.int64)
    flags = torch.zeros(n, dtype=torch.uint8, device=dev); flags[rows] = 1
    full = torch.zeros((n, 9), dtype=torch.float64, device=dev); full[rows] = g2d; mark("scatter")
    R._chain(cloud, cam, flags, full); mark("chain")
    torch.cuda.synchronize()
    print({tag: round(ev[i - 1][1].elapsed_time(e), 3) for i, (tag, e) in enumerate(ev) if i})
