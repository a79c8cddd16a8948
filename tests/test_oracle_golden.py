"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  No GPU needed."""

import numpy as np
import pytest

from helpers import intr_from, np_map, rel_err, window_maps, pose_from
from oracle import raster as O

I3 = np.eye(3)
Z3 = np.zeros(3)


def test_c1_projection_sort_tiles(golden):
    g = golden("c1")
    intr = intr_from(g["intr"])
    m = np_map(g, "in_", intr)
    b = O.prepare([m], I3, Z3, intr, learnable=0)
    np.testing.assert_array_equal(b.pixel_index, g["b_pixel"])
    np.testing.assert_array_equal(b.u0, g["b_u0"])
    np.testing.assert_array_equal(b.v0, g["b_v0"])
    np.testing.assert_array_equal(b.z, g["b_z"])
    # exp is restated (sgad_exp) and may differ from numpy's SIMD exp by 1 ulp
    np.testing.assert_allclose(b.sigma, g["b_sigma"], rtol=1e-15, atol=0)
    np.testing.assert_allclose(b.opacity, g["b_opacity"], rtol=1e-15, atol=0)
    off, lst = O.tile_lists(b)
    np.testing.assert_array_equal(off, g["offsets"])
    np.testing.assert_array_equal(lst, g["lists"])


def test_c1_loss_render_grads_adam(golden):
    g = golden("c1")
    intr = intr_from(g["intr"])
    m = np_map(g, "in_", intr)
    loss, grads, out = O.mapping_loss([m], g["t_color"], g["t_depth"], g["t_mask"], I3, Z3, intr)
    np.testing.assert_allclose([loss.total, loss.color_l1, loss.depth_l1],
                               g["loss"][[0, 1, 3]], rtol=1e-12)
    np.testing.assert_allclose(out.color, g["out_color"], atol=1e-12)
    np.testing.assert_allclose(out.depth, g["out_depth"], atol=1e-12)
    np.testing.assert_allclose(out.alpha, g["out_alpha"], atol=1e-12)
    np.testing.assert_array_equal(out.contributors, g["out_count"])
    for k, r in (("color", "g_color"), ("radius", "g_radius"), ("opacity_logit", "g_logit"),
                 ("delta", "g_delta")):
        assert rel_err(getattr(grads, k), g[r]) < 1e-9, k
    opt = O.Adam(m)
    opt.step(grads)
    for k, r in (("color", "adam_color"), ("log_radius", "adam_log_radius"),
                 ("opacity_logit", "adam_logit"), ("delta", "adam_delta")):
        np.testing.assert_allclose(getattr(m, k), g[r], atol=1e-12)


@pytest.mark.parametrize("view", [0, 2])
def test_window_views(golden, view):
    g = golden("window")
    intr, maps = window_maps(g)
    pose = pose_from(g[f"m{view}_pose"])
    b = O.prepare(maps, pose.rotation, pose.translation, intr, learnable="all")
    np.testing.assert_array_equal(b.pixel_index, g[f"v{view}_b_pixel"])
    np.testing.assert_array_equal(b.z, g[f"v{view}_b_z"])
    off, lst = O.tile_lists(b)
    np.testing.assert_array_equal(off, g[f"v{view}_offsets"])
    np.testing.assert_array_equal(lst, g[f"v{view}_lists"])
    out = O.forward(b, off, lst)
    np.testing.assert_allclose(out.color, g[f"v{view}_color"], atol=1e-12)
    np.testing.assert_allclose(out.depth, g[f"v{view}_depth"], atol=1e-12)
    np.testing.assert_array_equal(out.contributors, g[f"v{view}_count"])
    gc, gd, ga = g[f"v{view}_gc"], g[f"v{view}_gd"], g[f"v{view}_ga"]
    # delta D1: one all-learnable sweep + per-map chain == per-map splat_backward
    grads = O.splat_backward(maps, pose.rotation, pose.translation, intr, gc, gd, ga,
                             learnable_map="all")
    for i, gr in enumerate(grads):
        for k, r in (("color", "g_color"), ("radius", "g_radius"), ("opacity_logit", "g_logit"),
                     ("delta", "g_delta")):
            assert rel_err(getattr(gr, k), g[f"v{view}_m{i}_{r}"]) < 1e-9, (i, k)
    gn = O.splat_backward(maps, pose.rotation, pose.translation, intr, gc, gd, ga,
                          learnable_map=1, normalize_depth=True)
    assert rel_err(gn.delta, g[f"v{view}_norm_m1_g_delta"]) < 1e-9
    assert rel_err(gn.radius, g[f"v{view}_norm_m1_g_radius"]) < 1e-9
    outn = O.splat(maps, pose.rotation, pose.translation, intr, normalize_depth=True)
    np.testing.assert_allclose(outn.depth, g[f"v{view}_norm_depth"], atol=1e-12)
