"""The hand-written radix sort (csrc/radix.cu) against numpy's stable sort:
2-, 4- and 8-byte keys over arbitrary bit ranges [b0, b1) with nonzero bits
outside the range, ragged and empty inputs, unaligned arrays (the scalar
load paths), and the device-side item count of isg_sort_pairs_dev.  The
result of a stable sort is unique, so both placement schemes (reduce-then-scan
passes and the single-pass look-back) must produce exactly these arrays."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

DT = {2: (np.uint16, torch.int16), 4: (np.uint32, torch.int32), 8: (np.uint64, torch.int64)}


def _want(keys, vals, b0, b1):
    k = keys.astype(np.uint64)
    d = (k >> np.uint64(b0)) & np.uint64((1 << (b1 - b0)) - 1)
    o = np.argsort(d, kind="stable")
    return keys[o], vals[o]


def _sort(kb, keys, vals, b0, b1, n_dev=None, offset=0):
    from paper_2509_05216_b200 import _lib as L
    lib = L.lib()
    n = keys.shape[0]
    npt, tt = DT[kb]
    dev = torch.device("cuda", 0)
    # optional misalignment: the arrays start `offset` elements into a buffer
    kin = torch.zeros(n + offset + 1, dtype=tt, device=dev)
    vin = torch.zeros(n + offset + 1, dtype=torch.int32, device=dev)
    kin[offset:offset + n] = torch.from_numpy(keys.view(npt).astype(npt).view(np.int16 if kb == 2 else np.int32 if kb == 4 else np.int64))
    vin[offset:offset + n] = torch.from_numpy(vals)
    kout = torch.zeros(n + 1, dtype=tt, device=dev)
    vout = torch.zeros(n + 1, dtype=torch.int32, device=dev)
    p = lambda t, off=0: ctypes.c_void_p(t.data_ptr() + off * t.element_size())
    ws_bytes = ctypes.c_size_t(0)
    nd = None
    if n_dev is not None:
        nd = torch.tensor([n_dev], dtype=torch.int64, device=dev)
        f = lambda ws: lib.isg_sort_pairs_dev(ws, ctypes.byref(ws_bytes), kb, p(kin, offset), p(kout),
                                              p(vin, offset), p(vout), n, p(nd), b0, b1, L.stream_ptr())
    else:
        fn = {2: lib.isg_sort_u16, 4: lib.isg_sort_u32, 8: lib.isg_sort_u64}[kb]
        f = lambda ws: fn(ws, ctypes.byref(ws_bytes), p(kin, offset), p(kout), p(vin, offset), p(vout),
                          n, b0, b1, L.stream_ptr())
    L.check(f(None), "ws query")
    ws = torch.empty(max(int(ws_bytes.value), 1), dtype=torch.uint8, device=dev)
    L.check(f(ctypes.c_void_p(ws.data_ptr())), "sort")
    torch.cuda.synchronize()
    m = n if n_dev is None else n_dev
    ko = kout[:m].cpu().numpy().view(npt)
    vo = vout[:m].cpu().numpy()
    return ko, vo


@pytest.mark.parametrize("kb", [2, 4, 8])
@pytest.mark.parametrize("n", [0, 1, 1023, 1024, 2049, 100_003, 3_000_017])
def test_sort_matches_stable_argsort(kb, n):
    npt, _ = DT[kb]
    rng = np.random.default_rng(n + kb)
    keys = rng.integers(0, np.iinfo(npt).max, n, dtype=npt, endpoint=True)
    keys[: n // 3] &= npt(0x0F0F)  # many equal digits
    vals = np.arange(n, dtype=np.int32)
    for b0, b1 in ((0, 8 * kb), (3, 8 * kb - 2), (1, 12 if kb > 1 else 9)):
        got_k, got_v = _sort(kb, keys, vals, b0, b1)
        want_k, want_v = _want(keys, vals, b0, b1)
        np.testing.assert_array_equal(got_v, want_v, err_msg=f"vals {b0}-{b1}")
        np.testing.assert_array_equal(got_k, want_k, err_msg=f"keys {b0}-{b1}")


@pytest.mark.parametrize("kb", [2, 4, 8])
def test_sort_unaligned_and_device_count(kb):
    npt, _ = DT[kb]
    n = 500_001
    rng = np.random.default_rng(kb)
    keys = rng.integers(0, 1 << 14, n, dtype=npt)
    vals = rng.permutation(n).astype(np.int32)
    got_k, got_v = _sort(kb, keys, vals, 0, 14, offset=1)
    want_k, want_v = _want(keys, vals, 0, 14)
    np.testing.assert_array_equal(got_v, want_v)
    np.testing.assert_array_equal(got_k, want_k)
    m = 333_333
    got_k, got_v = _sort(kb, keys, vals, 0, 14, n_dev=m)
    want_k, want_v = _want(keys[:m], vals[:m], 0, 14)
    np.testing.assert_array_equal(got_v, want_v)
    np.testing.assert_array_equal(got_k, want_k)
