"""The reference's rasterizer known-answer tests (raysplat tests/test_rasterizer.py
TestForward :26-143 and TestBackward :222-275), restated against the drop-in
`splat` / `splat_backward` on the GPU: closed-form composites, ordering and
tie rules, the transmittance cutoff and alpha clamp, culling, depth
normalisation, and finite-difference gradient checks.  The scenes are
rebuilt here from their descriptions (pixel-aligned single-column layers,
a fronto-parallel plane, a three-Gaussian source map)."""

from types import SimpleNamespace

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2603_21055_b200.gaussians import init_gaussians
from paper_2603_21055_b200.geometry import Intrinsics, Pose, se3_exp
from paper_2603_21055_b200.rasterizer import splat, splat_backward


def row_camera(width, f=50.0):
    """A 1-pixel-high camera: column u looks along ((u - cx) / f, 0, 1)."""
    return Intrinsics(fx=f, fy=f, cx=(width - 1) / 2.0, cy=0.0, width=width, height=1)


def layer_maps(alphas, colors, depths, intr):
    """One 1 x W map per layer j, at constant depth depths[j], opacity
    alphas[j][u] and colour colors[j][u]; radius 0.05 px so every Gaussian
    covers only its own pixel column of the (identity) target camera."""
    maps = []
    w = intr.width
    for j, z in enumerate(depths):
        base = np.full((1, w), float(z))
        frame = SimpleNamespace(depth=base, color=np.asarray(colors[j], float).reshape(1, w, 3),
                                intrinsics=intr, index=j)
        m = init_gaussians(frame, Pose.identity(), base_depth=base)
        a = np.asarray(alphas[j], float).reshape(1, w)
        m.log_radius[:] = torch.from_numpy(np.log(np.full((1, w), 0.05 * z / intr.fx)))
        with np.errstate(divide="ignore"):
            m.opacity_logit[:] = torch.from_numpy(np.log(a / (1.0 - a)))
        maps.append(m)
    return maps


def composite_ray(alphas, colors, depths):
    """Front-to-back over one ray, layers given in depth order (no cutoff)."""
    c, d, a, t = np.zeros(3), 0.0, 0.0, 1.0
    for al, col, z in zip(alphas, colors, depths):
        c = c + np.asarray(col) * al * t
        d += z * al * t
        a += al * t
        t *= 1.0 - al
    return c, d, a


def plane_frame(depth=0.9, w=64, h=48, fx=100.0, color=(0.6, 0.4, 0.3)):
    """A fronto-parallel plane filling the view at `depth`."""
    intr = Intrinsics(fx=fx, fy=fx, cx=(w - 1) / 2, cy=(h - 1) / 2, width=w, height=h)
    return SimpleNamespace(depth=np.full((h, w), depth), color=np.broadcast_to(color, (h, w, 3)).copy(),
                           intrinsics=intr, index=0)


def np_(t):
    return t.detach().cpu().numpy() if torch.is_tensor(t) else np.asarray(t)


# ------------------------------------------------------------------ forward

def test_no_sources_renders_zeros():
    out = splat([], Pose.identity(), row_camera(4))
    assert not np_(out.color).any() and not np_(out.alpha).any() and not np_(out.contributors).any()


def test_one_layer_half_opacity():
    intr = row_camera(3)
    out = splat(layer_maps([[0.5] * 3], [[(1.0, 0.5, 0.25)] * 3], [2.0], intr), Pose.identity(), intr)
    np.testing.assert_allclose(np_(out.color)[0, 1], [0.5, 0.25, 0.125], atol=1e-12)
    np.testing.assert_allclose(np_(out.depth)[0, 1], 1.0, atol=1e-12)
    np.testing.assert_allclose(np_(out.alpha)[0, 1], 0.5, atol=1e-12)
    assert np_(out.contributors)[0, 1] == 1


def test_two_layers_closed_form():
    intr = row_camera(1)
    maps = layer_maps([[0.5], [0.5]], [[(1.0, 0.0, 0.0)], [(0.0, 1.0, 0.0)]], [1.0, 2.0], intr)
    out = splat(maps, Pose.identity(), intr)
    np.testing.assert_allclose(np_(out.color)[0, 0], [0.5, 0.25, 0.0], atol=1e-12)
    np.testing.assert_allclose(np_(out.depth)[0, 0], 0.5 + 0.5, atol=1e-12)
    np.testing.assert_allclose(np_(out.alpha)[0, 0], 0.75, atol=1e-12)


def test_random_stacks_match_ray_composite():
    rng = np.random.default_rng(0)
    intr = row_camera(32)
    depths = [0.8, 1.3, 1.9, 2.6]
    alphas = [rng.uniform(0.05, 0.9, 32) for _ in depths]
    colors = [rng.uniform(0.0, 1.0, (32, 3)) for _ in depths]
    out = splat(layer_maps(alphas, colors, depths, intr), Pose.identity(), intr)
    for u in range(32):
        c, d, a = composite_ray([x[u] for x in alphas], [x[u] for x in colors], depths)
        np.testing.assert_allclose(np_(out.color)[0, u], c, atol=1e-12)
        np.testing.assert_allclose(np_(out.depth)[0, u], d, atol=1e-12)
        np.testing.assert_allclose(np_(out.alpha)[0, u], a, atol=1e-12)


def test_map_order_does_not_matter():
    rng = np.random.default_rng(1)
    intr = row_camera(16)
    depths = [1.0, 1.5, 2.0]
    maps = layer_maps([rng.uniform(0.1, 0.9, 16) for _ in depths],
                      [rng.uniform(0.0, 1.0, (16, 3)) for _ in depths], depths, intr)
    a = splat(maps, Pose.identity(), intr)
    b = splat(maps[::-1], Pose.identity(), intr)
    np.testing.assert_array_equal(np_(a.color), np_(b.color))
    np.testing.assert_array_equal(np_(a.depth), np_(b.depth))


def test_equal_depths_composite_in_frame_order():
    intr = row_camera(1)
    maps = layer_maps([[0.8], [0.4]], [[(1.0, 0.0, 0.0)], [(0.0, 1.0, 0.0)]], [1.5, 1.5], intr)
    out = splat(maps, Pose.identity(), intr)
    np.testing.assert_allclose(np_(out.color)[0, 0, 0], 0.8, atol=1e-12)  # frame 0 first
    np.testing.assert_allclose(np_(out.color)[0, 0, 1], 0.4 * 0.2, atol=1e-12)
    np.testing.assert_array_equal(np_(splat(maps[::-1], Pose.identity(), intr).color), np_(out.color))


def test_stops_after_transmittance_cutoff():
    # alpha 0.95 per layer: T = 0.05^k drops below 1e-4 with the 4th layer
    intr = row_camera(1)
    n = 50
    maps = layer_maps([[0.95]] * n, [[(1.0, 1.0, 1.0)]] * n, list(1.0 + 0.05 * np.arange(n)), intr)
    out = splat(maps, Pose.identity(), intr)
    assert np_(out.contributors)[0, 0] == 4
    assert np_(out.alpha)[0, 0] < 1.0


def test_alpha_clamped_at_0999():
    intr = row_camera(1)
    out = splat(layer_maps([[0.9999]], [[(1.0, 1.0, 1.0)]], [1.0], intr), Pose.identity(), intr)
    np.testing.assert_allclose(np_(out.alpha)[0, 0], 0.999, atol=1e-9)


def test_opaque_map_reprojects_its_own_depth():
    f = plane_frame(depth=0.9)
    m = init_gaussians(f, Pose.identity())
    m.opacity_logit[:] = 20.0
    out = splat([m], Pose.identity(), f.intrinsics)
    err = np.abs(np_(out.depth) - f.depth)[4:-4, 4:-4]
    assert err.max() <= 1e-4


def test_points_behind_the_camera_are_culled():
    f = plane_frame(depth=0.9)
    m = init_gaussians(f, Pose.identity())
    out = splat([m], Pose(np.eye(3), np.array([0.0, 0.0, 2.0])), f.intrinsics)
    assert not np_(out.alpha).any()


def test_normalised_depth():
    intr = row_camera(1)
    maps = layer_maps([[0.5], [0.5]], [[(1.0, 0.0, 0.0)], [(0.0, 1.0, 0.0)]], [1.0, 2.0], intr)
    out = splat(maps, Pose.identity(), intr, normalize_depth=True)
    np.testing.assert_allclose(np_(out.depth)[0, 0], (0.5 + 0.5) / 0.75, atol=1e-12)


def test_accumulated_alpha_in_unit_range():
    f = plane_frame()
    m = init_gaussians(f, Pose.identity())
    m.opacity_logit[:] = 8.0
    a = np_(splat([m], Pose.identity(), f.intrinsics).alpha)
    assert a.max() <= 1.0 + 1e-12 and a.min() >= 0.0


# ------------------------------------------------------------------ backward

def test_zero_upstream_zero_gradients():
    f = plane_frame(w=16, h=16)
    m = init_gaussians(f, Pose.identity())
    z = np.zeros((16, 16))
    g = splat_backward([m], Pose.identity(), f.intrinsics, np.zeros((16, 16, 3)), z, z)
    for k in ("color", "radius", "opacity_logit", "delta"):
        assert not np_(getattr(g, k)).any(), k


def test_colour_gradient_of_one_layer_is_its_alpha():
    intr = row_camera(3)
    maps = layer_maps([[0.5] * 3], [[(0.3, 0.3, 0.3)] * 3], [2.0], intr)
    gc = np.zeros((1, 3, 3))
    gc[0, 1, 0] = 1.0
    z = np.zeros((1, 3))
    g = np_(splat_backward(maps, Pose.identity(), intr, gc, z, z).color)
    np.testing.assert_allclose(g[0, 1, 0], 0.5, atol=1e-12)
    assert g[0, 0, 0] == 0.0 and g[0, 2, 0] == 0.0


def test_occluded_layer_sees_front_transmittance():
    intr = row_camera(4)
    maps = layer_maps([[0.5] * 4, [0.6] * 4], [[(0.2, 0.4, 0.6)] * 4, [(0.8, 0.1, 0.3)] * 4],
                      [1.0, 1.6], intr)
    ones = np.ones((1, 4))
    g0 = np_(splat_backward(maps, Pose.identity(), intr, np.ones((1, 4, 3)), ones, ones,
                            learnable_map=0).color)
    g1 = np_(splat_backward(maps, Pose.identity(), intr, np.ones((1, 4, 3)), ones, ones,
                            learnable_map=1).color)
    assert np.abs(g0).max() > 0.0 and np.abs(g1).max() > 0.0
    np.testing.assert_allclose(g1[0, 0], 0.6 * 0.5, atol=1e-12)


def test_gaussians_out_of_view_get_zero_gradient():
    f = plane_frame(w=16, h=16)
    m = init_gaussians(f, Pose.identity())
    ones = np.ones((16, 16))
    g = splat_backward([m], se3_exp([0.0, 1.2, 0.0, 0.0, 0.0, 0.0]), f.intrinsics,
                       np.ones((16, 16, 3)), ones, ones)
    assert not np_(g.delta).any()


def three_gaussians(rng):
    """A 3-pixel source map seen by a 16x16 camera from a small random pose,
    drawn away from the model's kinks (3-sigma edges, the alpha clamp, the
    cutoff, |base + delta| = 0) so central differences are a valid check."""
    tgt = Intrinsics(fx=30.0, fy=30.0, cx=7.5, cy=7.5, width=16, height=16)
    src = Intrinsics(fx=30.0, fy=30.0, cx=1.0, cy=0.0, width=3, height=1)
    while True:
        base = rng.uniform(0.8, 1.2, (1, 3))
        frame = SimpleNamespace(depth=base, color=rng.uniform(0.1, 0.9, (1, 3, 3)), intrinsics=src,
                                index=0)
        m = init_gaussians(frame, Pose.identity(), base_depth=base)
        m.delta[:] = torch.from_numpy(rng.uniform(-0.05, 0.05, (1, 3)))
        m.log_radius[:] = torch.from_numpy(np.log(rng.uniform(0.04, 0.12, (1, 3))))
        m.opacity_logit[:] = torch.from_numpy(rng.uniform(-1.5, 2.2, (1, 3)))
        pose = se3_exp(np.concatenate([rng.uniform(-0.03, 0.03, 3), rng.uniform(-0.02, 0.02, 3)]))
        if fd_safe(m, pose, tgt):
            return m, pose, tgt


def fd_safe(m, pose, tgt, margin=0.05):
    rel = pose.inverse().compose(m.pose)
    src = m.intrinsics
    d = np_(m.adjusted_depth)[0]
    r = np_(m.radius)[0]
    uu, vv = np.meshgrid(np.arange(tgt.width), np.arange(tgt.height))
    for j in range(3):
        y = rel.rotation @ np.array([(j - src.cx) / src.fx, (0 - src.cy) / src.fy, 1.0]) * d[j] \
            + rel.translation
        if y[2] <= 1e-3:
            return False
        u0, v0 = tgt.fx * y[0] / y[2] + tgt.cx, tgt.fy * y[1] / y[2] + tgt.cy
        if not (2.0 < u0 < tgt.width - 3.0 and 2.0 < v0 < tgt.height - 3.0):
            return False
        if np.abs(np.hypot(uu - u0, vv - v0) - 3.0 * r[j] * tgt.fx / y[2]).min() < margin:
            return False
    return True


def worst_fd_error(rng, normalize_depth):
    m, pose, intr = three_gaussians(rng)
    gc, gd, ga = rng.normal(size=(16, 16, 3)), rng.normal(size=(16, 16)), rng.normal(size=(16, 16))
    g = splat_backward([m], pose, intr, gc, gd, ga, learnable_map=0, normalize_depth=normalize_depth)

    def loss():
        o = splat([m], pose, intr, normalize_depth=normalize_depth)
        return float((np_(o.color) * gc).sum() + (np_(o.depth) * gd).sum() + (np_(o.alpha) * ga).sum())

    worst = 0.0

    def check(analytic, read, write):
        nonlocal worst
        v = read()
        h = 1e-4 * max(1.0, abs(v))
        write(v + h)
        lp = loss()
        write(v - h)
        lm = loss()
        write(v)
        fd = (lp - lm) / (2 * h)
        worst = max(worst, abs(fd - analytic) / max(abs(fd), abs(analytic), 1e-4))

    P = m.planes  # [7, 1, 3]: base, delta, log radius, logit, R, G, B
    gcol, grad, glog, gdel = (np_(x) for x in (g.color, g.radius, g.opacity_logit, g.delta))
    for j in range(3):
        for c in range(3):
            check(gcol[0, j, c], lambda: float(P[4 + c, 0, j]),
                  lambda x, c=c, j=j: P[4 + c, 0, j].fill_(x))
        # the radius gradient is with respect to r itself (mapper.py:77 chains it)
        check(grad[0, j], lambda j=j: float(torch.exp(P[2, 0, j])),
              lambda x, j=j: P[2, 0, j].fill_(float(np.log(x))))
        check(glog[0, j], lambda j=j: float(P[3, 0, j]), lambda x, j=j: P[3, 0, j].fill_(x))
        check(gdel[0, j], lambda j=j: float(P[1, 0, j]), lambda x, j=j: P[1, 0, j].fill_(x))
    return worst


def test_gradients_match_central_differences():
    rng = np.random.default_rng(42)
    for _ in range(20):
        assert worst_fd_error(rng, normalize_depth=False) < 1e-3


def test_normalised_depth_gradients_match_central_differences():
    rng = np.random.default_rng(43)
    for _ in range(5):
        assert worst_fd_error(rng, normalize_depth=True) < 1e-3
