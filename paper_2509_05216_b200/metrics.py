"""Training loss and evaluation metrics (reference metrics.py) on B200 kernels.

loss_l1_dssim is the fused two-pass stencil of csrc/loss.cu (compute type =
image dtype); ssim runs the same field pass in float64; psnr is a reduction.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _lib as L

PSNR_CAP = 100.0
SSIM_WINDOW = 11

_WS = L.Workspace()


def _dev(x, dtype=None) -> torch.Tensor:
    dev = L.require_cuda()
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(dev).contiguous()


def loss_l1_dssim_device(img: torch.Tensor, ref: torch.Tensor, lambda_dssim: float,
                         grad: torch.Tensor, loss_out: torch.Tensor) -> None:
    """Stream-ordered core: writes dL/dimg into `grad` and the loss into
    loss_out[0] (float64, device) without a host sync."""
    h, w = int(img.shape[0]), int(img.shape[1])
    sz = ctypes.c_size_t(0)
    tag = L.dtype_tag(img.dtype)
    u8 = 1 if ref.dtype == torch.uint8 else 0
    if not u8 and ref.dtype != img.dtype:
        raise ValueError("ref must match the image dtype or be uint8 codes")
    L.check(L.lib().isg_loss_l1_dssim(None, ctypes.byref(sz), tag, h, w, None, None, u8,
                                      float(lambda_dssim), None, None, None), "loss (size)")
    buf = _WS.get(sz.value, img.device)
    sz = ctypes.c_size_t(buf.numel())
    L.check(L.lib().isg_loss_l1_dssim(L.ptr(buf), ctypes.byref(sz), tag, h, w, L.ptr(img),
                                      L.ptr(ref), u8, float(lambda_dssim), L.ptr(grad),
                                      L.ptr(loss_out), L.stream_ptr()), "isg_loss_l1_dssim")


def loss_l1_dssim(img, ref, lambda_dssim: float = 0.2):
    """(1 - lam) * L1 + lam * (1 - SSIM) and its image gradient
    (metrics.py:135-189).  Returns (float, grad in img's dtype)."""
    if not 0.0 <= lambda_dssim <= 1.0:
        raise ValueError("lambda_dssim must lie in [0, 1]")
    a = _dev(img)
    if a.dtype not in (torch.float32, torch.float64):
        a = a.to(torch.float64)
    b = _dev(ref, a.dtype)
    if a.shape != b.shape or a.ndim != 3 or a.shape[2] != 3:
        raise ValueError(f"expected matching (H, W, 3) images, got {tuple(a.shape)} vs {tuple(b.shape)}")
    h, w = a.shape[:2]
    if h < SSIM_WINDOW or w < SSIM_WINDOW:
        raise ValueError(f"image {h}x{w} smaller than the {SSIM_WINDOW}x{SSIM_WINDOW} SSIM window")
    grad = torch.empty_like(a)
    loss = torch.empty(1, dtype=torch.float64, device=a.device)
    loss_l1_dssim_device(a, b, lambda_dssim, grad, loss)
    return float(loss.item()), grad


def ssim(img, ref) -> float:
    """Mean SSIM over valid centres, averaged over channels (metrics.py:127-132)."""
    a = _dev(img, torch.float64)
    b = _dev(ref, torch.float64)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {tuple(a.shape)} vs {tuple(b.shape)}")
    if a.ndim == 2:
        a = a[:, :, None].contiguous()
        b = b[:, :, None].contiguous()
    if a.ndim != 3:
        raise ValueError(f"expected (H, W) or (H, W, C), got {tuple(a.shape)}")
    h, w, c = (int(v) for v in a.shape)
    if h < SSIM_WINDOW or w < SSIM_WINDOW:
        raise ValueError(f"image {h}x{w} smaller than the {SSIM_WINDOW}x{SSIM_WINDOW} SSIM window")
    sz = ctypes.c_size_t(0)
    L.check(L.lib().isg_ssim(None, ctypes.byref(sz), h, w, c, None, None, None, None), "ssim (size)")
    buf = _WS.get(sz.value, a.device)
    sz = ctypes.c_size_t(buf.numel())
    out = torch.empty(1, dtype=torch.float64, device=a.device)
    L.check(L.lib().isg_ssim(L.ptr(buf), ctypes.byref(sz), h, w, c, L.ptr(a), L.ptr(b),
                             L.ptr(out), L.stream_ptr()), "isg_ssim")
    return float(out.item())


def psnr(img, ref) -> float:
    """PSNR in dB for [0, 1] images, capped at 100 (metrics.py:75-84)."""
    a = _dev(img, torch.float64)
    b = _dev(ref, torch.float64)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {tuple(a.shape)} vs {tuple(b.shape)}")
    mse = float(torch.mean((a - b) ** 2).item())
    if mse == 0.0:
        return PSNR_CAP
    return min(-10.0 * math.log10(mse), PSNR_CAP)


def quantize8(img: torch.Tensor) -> torch.Tensor:
    """images.py:9-16: clamp to [0, 1], round half-to-even on the 8-bit grid."""
    return torch.round(torch.clamp(img.to(torch.float64), 0.0, 1.0) * 255.0) / 255.0
