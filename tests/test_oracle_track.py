"""Pin the tracking oracle (window fit + GICP restatement) against golden
vectors produced by the reference (tests/golden/make_golden.py)."""

import numpy as np

from oracle import track as OT


def test_eig_matches_reference(golden):
    g = golden("eig")
    rot, vals = OT.sym_eigh3_batch(g["mats"])
    np.testing.assert_allclose(vals, g["vals"], atol=1e-12)
    np.testing.assert_allclose(rot, g["rot"], atol=1e-9)


def _fit(g, name):
    fx, fy, cx, cy = g["intr"][:4]
    return OT.window_fit(g[f"{name}_depth"], g[f"{name}_mask"], fx, fy, cx, cy)


def test_window_fit_matches_reference(golden):
    g = golden("track")
    for name in ("ref", "qry"):
        idx, c, rot, s, n = _fit(g, name)
        np.testing.assert_array_equal(idx, g[f"{name}_idx"])
        np.testing.assert_array_equal(c, g[f"{name}_centers"])
        np.testing.assert_allclose(n, g[f"{name}_normals"], atol=1e-9)
        np.testing.assert_allclose(s, g[f"{name}_scales"], atol=1e-9)
        np.testing.assert_allclose(OT.covariances(rot, s),
                                   OT.covariances(g[f"{name}_rot"], g[f"{name}_scales"]),
                                   atol=1e-12)


def test_gicp_matches_reference(golden):
    g = golden("track")
    lc, lr, ls = g["qry_centers"], g["qry_rot"], g["qry_scales"]
    gc, gr, gs, gn = g["ref_centers"], g["ref_rot"], g["ref_scales"], g["ref_normals"]
    R, t, d = OT.gicp_align(lc, OT.covariances(lr, ls), gc, OT.covariances(gr, gs), gn,
                            np.eye(3), np.zeros(3), max_iters=20, eps=0.0)
    assert d.iterations == int(g["gicp_iters"])
    assert d.inlier_count == int(g["gicp_inliers"])
    np.testing.assert_array_equal(d.accepted_first, g["gicp_accepted_first"])
    np.testing.assert_allclose(np.concatenate([R.reshape(9), t]), g["gicp_pose"], atol=1e-12)
    np.testing.assert_allclose(np.array(d.cost_pairs), g["gicp_cost_pairs"], rtol=1e-9)
    h, gg, c, _ = d.systems[0]
    np.testing.assert_allclose(h, g["first_H"], rtol=1e-12, atol=1e-12 * np.abs(g["first_H"]).max())
    np.testing.assert_allclose(gg, g["first_g"], rtol=1e-12, atol=1e-12 * np.abs(g["first_g"]).max())
