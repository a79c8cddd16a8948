"""Windowed SSIM with the gradient w.r.t. the first image, on the GPU.

Drop-in for ``raysplat/ssim.py:31-87`` (``ssim(img_a, img_b, with_grad)``):
11x11 Gaussian window (sigma 1.5), zero padding with the window mass
renormalised over the in-bounds support, C1 = 0.01^2, C2 = 0.03^2, mean over
pixels and channels.  Computed by ``sgad_ssim`` (csrc/ssim.cu) in fp64.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native as N

SSIM_C1 = 0.01**2
SSIM_C2 = 0.03**2


def _as_image(x, device, dtype=torch.float64):
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x))
    return t.to(device=device, dtype=dtype).contiguous()


def workspace_bytes(h: int, w: int, c: int) -> int:
    n = ctypes.c_int64()
    N.check(N.load().sgad_ssim_workspace_size(int(h), int(w), int(c), ctypes.byref(n)))
    return n.value


def ssim_sum(img_a: torch.Tensor, img_b: torch.Tensor, sum_out: torch.Tensor, grad_out=None,
             workspace=None, kc: float = 0.0, tau: float = 0.0, upstream: bool = False,
             stream=None) -> None:
    """Low-level entry: device [H, W, C] images (a fp64, b fp64 or fp32);
    ``sum_out`` (device fp64 scalar) += sum of per-pixel SSIM; optional
    gradient / loss upstream into ``grad_out`` (see include/sgad.h)."""
    h, w, c = img_a.shape
    N.check(N.load().sgad_ssim(N.ptr(img_a), N.ptr(img_b), int(img_b.dtype == torch.float32),
                               int(h), int(w), int(c), N.ptr(sum_out), N.ptr(grad_out),
                               N.ptr(workspace), float(kc), float(tau), int(upstream),
                               N.stream_ptr(stream)))


def ssim(img_a, img_b, with_grad: bool = False, device=None):
    """ssim.py:31-87.  Accepts (H, W) or (H, W, C) arrays/tensors in [0, 1];
    returns the mean SSIM, or ``(value, grad)`` with ``grad`` a device fp64
    tensor shaped like ``img_a``."""
    dev = torch.device(device) if device is not None else (
        img_a.device if isinstance(img_a, torch.Tensor) and img_a.is_cuda
        else torch.device("cuda", torch.cuda.current_device()))
    a = _as_image(img_a, dev)
    b = _as_image(img_b, dev)
    if a.shape != b.shape:
        raise ValueError(f"image shapes differ: {tuple(a.shape)} vs {tuple(b.shape)}")
    squeeze = a.dim() == 2
    if squeeze:
        a, b = a[:, :, None].contiguous(), b[:, :, None].contiguous()
    h, w, c = a.shape
    total = torch.zeros((), dtype=torch.float64, device=dev)
    grad = ws = None
    if with_grad:
        grad = torch.empty_like(a)
        ws = torch.empty(max(workspace_bytes(h, w, c) // 8, 1), dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        ssim_sum(a, b, total, grad, ws)
    value = float(total) / float(a.numel())
    if not with_grad:
        return value
    return value, (grad[:, :, 0] if squeeze else grad)
