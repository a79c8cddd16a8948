"""Hole-free depth for Gaussian placement -- drop-in for
raysplat/datasets.py:368-398 (``inpaint_depth``): holes are seeded with their
nearest valid value (scipy's Euclidean distance transform on the host, the
reference's own call) and relaxed by Jacobi sweeps of the grid Laplace
equation on the GPU (``sgad_inpaint_jacobi``, bit-identical to the
reference's numpy loop)."""

from __future__ import annotations

import ctypes

import numpy as np
import torch
from scipy import ndimage

from . import _native as N


def inpaint_depth(depth, valid_mask, max_iters: int = 200, tol: float = 1e-5,
                  return_sweeps: bool = False):
    """datasets.py:368-398: fill invalid depth by harmonic diffusion from the
    valid pixels; a fully valid input is returned unchanged (idempotent)."""
    d = depth.detach().cpu().numpy() if isinstance(depth, torch.Tensor) else depth
    d = np.asarray(d, dtype=np.float64)
    m = valid_mask.detach().cpu().numpy() if isinstance(valid_mask, torch.Tensor) else valid_mask
    valid = np.asarray(m, dtype=bool) & (d > 0)
    if not valid.any():
        raise ValueError("cannot inpaint a frame with no valid depth")
    if valid.all():
        return (d.copy(), 0) if return_sweeps else d.copy()
    _, (iy, ix) = ndimage.distance_transform_edt(~valid, return_indices=True)
    seed = d[iy, ix]
    seed[valid] = d[valid]
    dev = torch.device("cuda", torch.cuda.current_device())
    out = torch.as_tensor(seed, device=dev).contiguous()
    hole = torch.as_tensor((~valid).astype(np.uint8), device=dev).contiguous()
    scratch = torch.empty_like(out)
    sweeps = ctypes.c_int32()
    h, w = d.shape
    N.check(N.load().sgad_inpaint_jacobi(N.ptr(out), N.ptr(hole), int(h), int(w),
                                         int(max_iters), float(tol), N.ptr(scratch),
                                         ctypes.byref(sweeps), N.stream_ptr()))
    res = out.cpu().numpy()
    return (res, sweeps.value) if return_sweeps else res
