"""Dense Adam over named parameter groups (reference optim.py:12-64).

adam_step launches isg_adam per group; the float constants are rounded to the
storage dtype first, reproducing numpy's weak-scalar arithmetic bit for bit.
The training engine uses the fused isg_chain_adam instead (engine.py).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib as L

ADAM_BETA1 = 0.9
ADAM_BETA2 = 0.999
ADAM_EPS = 1e-15


def adam_init(params: dict) -> dict:
    """Zeroed first/second-moment buffers matching each parameter array."""
    return {name: {"m": torch.zeros_like(p), "v": torch.zeros_like(p)} for name, p in params.items()}


def adam_consts(dtype: torch.dtype, iteration: int, lr: float, beta1=ADAM_BETA1,
                beta2=ADAM_BETA2, eps=ADAM_EPS) -> L.AdamConsts_t:
    """optim.py:36-55 constants, rounded like numpy rounds a Python float
    operand to the array dtype."""
    bc1 = 1.0 - beta1 ** iteration
    bc2 = 1.0 - beta2 ** iteration
    r = (lambda x: float(np.float32(x))) if dtype == torch.float32 else float
    c = L.AdamConsts_t()
    c.b1, c.omb1, c.b2, c.omb2 = r(beta1), r(1.0 - beta1), r(beta2), r(1.0 - beta2)
    c.bc1, c.bc2, c.lr, c.eps = r(bc1), r(bc2), r(lr), r(eps)
    return c


def adam_step(params: dict, grads: dict, state: dict, iteration: int, lrs: dict,
              beta1: float = ADAM_BETA1, beta2: float = ADAM_BETA2, eps: float = ADAM_EPS):
    """One bias-corrected Adam update, in place, per group (optim.py:20-56)."""
    if iteration < 1:
        raise ValueError("iteration must be >= 1")
    for name, p in params.items():
        g = grads[name]
        if tuple(g.shape) != tuple(p.shape):
            raise ValueError(f"{name}: grad shape {tuple(g.shape)} != param shape {tuple(p.shape)}")
        st = state[name]
        m, v = st["m"], st["v"]
        if tuple(m.shape) != tuple(p.shape):
            raise ValueError(f"{name}: state shape {tuple(m.shape)} != param shape {tuple(p.shape)}")
        if not (p.is_cuda and p.is_contiguous() and m.is_contiguous() and v.is_contiguous()):
            raise ValueError(f"{name}: params and state must be contiguous CUDA tensors")
        g = g.to(device=p.device, dtype=p.dtype).contiguous()
        c = adam_consts(p.dtype, iteration, lrs[name], beta1, beta2, eps)
        L.check(L.lib().isg_adam(L.dtype_tag(p.dtype), p.numel(), L.ptr(p), L.ptr(g), L.ptr(m),
                                 L.ptr(v), ctypes.byref(c), L.stream_ptr()), "isg_adam")
    return params, state


def position_lr(base_lr: float, iteration: int, total: int, final_mult: float = 0.01) -> float:
    """Exponential decay from base_lr to final_mult * base_lr (optim.py:59-64)."""
    if total <= 0:
        return base_lr
    t = min(max(iteration, 0), total) / total
    return base_lr * (final_mult ** t)
