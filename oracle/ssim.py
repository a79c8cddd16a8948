"""CPU oracle (test infrastructure only) for the SSIM term of the mapping
objective, /root/reference/pkg/src/raysplat/ssim.py:31-87: local means,
variances and covariance under an 11x11 Gaussian window (sigma 1.5,
ssim.py:21-25), zero padding renormalised by the in-bounds window mass
(:48), C1 = 1e-4, C2 = 9e-4 (:16-17), and the analytic gradient of the mean
w.r.t. the first image (:73-81).  Third-party arithmetic: scipy.ndimage
(the reference's own dependency, scipy >= 1.10; 1.18.1 here), applied here
to all channels at once.  Pinned by tests/golden/ssim.npz, produced by the
reference itself (tests/golden/make_golden.py)."""

from __future__ import annotations

import numpy as np
from scipy import ndimage

_K1SQ, _K2SQ = 1e-4, 9e-4


def _kernel3(radius=5, sd=1.5):
    t = (np.arange(2 * radius + 1, dtype=np.float64) - radius) / sd
    w1 = np.exp(-0.5 * t**2)
    w2 = np.outer(w1, w1)
    return (w2 / w2.sum())[:, :, None]


def _filt(stack, ker):
    return ndimage.correlate(stack, ker, mode="constant", cval=0.0)


def ssim(img_a, img_b, with_grad=False):
    """Mean SSIM of two images in [0, 1] ((H, W) or (H, W, C)); with
    ``with_grad`` also d(mean)/d(img_a)."""
    x = np.atleast_3d(np.asarray(img_a, dtype=np.float64))
    y = np.atleast_3d(np.asarray(img_b, dtype=np.float64))
    ker = _kernel3()
    wsum = _filt(np.ones(x.shape[:2] + (1,)), ker)
    mu_x, mu_y = _filt(x, ker) / wsum, _filt(y, ker) / wsum
    var_x = _filt(x * x, ker) / wsum - mu_x**2
    var_y = _filt(y * y, ker) / wsum - mu_y**2
    cov = _filt(x * y, ker) / wsum - mu_x * mu_y
    num_l, num_c = 2.0 * mu_x * mu_y + _K1SQ, 2.0 * cov + _K2SQ
    den_l, den_c = mu_x**2 + mu_y**2 + _K1SQ, var_x + var_y + _K2SQ
    smap = num_l * num_c / (den_l * den_c)
    mean = float(smap.sum() / x.size)
    if not with_grad:
        return mean
    d_var = -smap / den_c
    d_cov = 2.0 * num_l / (den_l * den_c)
    d_mu = 2.0 * (mu_y * num_c / den_c - mu_x * smap) / den_l - 2.0 * mu_x * d_var - mu_y * d_cov
    g = (_filt(d_mu / wsum, ker) + 2.0 * x * _filt(d_var / wsum, ker)
         + y * _filt(d_cov / wsum, ker)) / x.size
    return mean, (g[:, :, 0] if np.ndim(img_a) == 2 else g)
