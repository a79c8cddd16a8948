"""Pin the SSIM oracle (oracle/ssim.py) and the tau != 0 mapping objective
against golden vectors produced by the reference (raysplat/ssim.py:31-87,
mapper.py:106-157).  No GPU needed."""

import numpy as np
import pytest

from helpers import intr_from, np_map, rel_err
from oracle import raster as O
from oracle import ssim as OS


@pytest.mark.parametrize("case", ["rgb", "gray", "const", "tiny"])
def test_ssim_value_and_grad(golden, case):
    g = golden("ssim")
    v, grad = OS.ssim(g[f"{case}_a"], g[f"{case}_b"], with_grad=True)
    assert abs(v - float(g[f"{case}_value"])) < 1e-13
    assert grad.shape == g[f"{case}_grad"].shape
    np.testing.assert_allclose(grad, g[f"{case}_grad"], rtol=0, atol=1e-15)
    assert OS.ssim(g[f"{case}_a"], g[f"{case}_b"]) == v


def test_ssim_identical_images_is_one():
    a = np.random.default_rng(1).random((20, 30, 3))
    v, grad = OS.ssim(a, a, with_grad=True)
    assert abs(v - 1.0) < 1e-12
    assert np.abs(grad).max() < 1e-12


def test_c1_tau_objective(golden):
    """tau = 0.2: the SSIM term enters the loss and the colour upstream."""
    g, s = golden("c1"), golden("ssim")
    intr = intr_from(g["intr"])
    m = np_map(g, "in_", intr)
    loss, grads, _ = O.mapping_loss([m], s["c1_t_color"], s["c1_t_depth"], s["c1_t_mask"],
                                    np.eye(3), np.zeros(3), intr, tau=0.2)
    np.testing.assert_allclose([loss.total, loss.color_l1, loss.ssim_term, loss.depth_l1],
                               s["c1_loss"], rtol=1e-12)
    for k, r in (("color", "c1_g_color"), ("radius", "c1_g_radius"),
                 ("opacity_logit", "c1_g_logit"), ("delta", "c1_g_delta")):
        assert rel_err(getattr(grads, k), s[r]) < 1e-9, k
