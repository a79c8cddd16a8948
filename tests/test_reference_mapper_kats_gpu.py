"""The reference's optimizer and mapping-objective known-answer tests
(raysplat tests/test_mapper.py TestOptimizer :69-131, TestMappingLoss
:148-235), restated against the drop-in MapOptimizer and mapping_loss on the
GPU: the first Adam step is -lr sign(g), zero gradients leave the map alone,
the offset can be frozen, colours stay in [0, 1], the radius gradient is
chained through the log; the loss of a perfect target is zero, the
breakdown composes as rho L1 + tau SSIM + sigma masked depth L1, a frame
without valid depth stays finite, and the assembled gradient matches
central differences of the total loss."""

from types import SimpleNamespace

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2603_21055_b200.mapper import MapOptimizer, MapperConfig, mapping_loss
from paper_2603_21055_b200.rasterizer import MapGradients, splat

from test_reference_kats_gpu import fd_safe, np_, three_gaussians


def zero_grads(m):
    h, w = m.shape
    return MapGradients(color=np.zeros((h, w, 3)), radius=np.zeros((h, w)),
                        opacity_logit=np.zeros((h, w)), delta=np.zeros((h, w)))


def host(m, name):
    return np_(getattr(m, name)).copy()


def test_first_adam_step_is_signed_learning_rate():
    m, _, _ = three_gaussians(np.random.default_rng(0))
    cfg = MapperConfig()
    before = host(m, "color")
    g = zero_grads(m)
    g.color[0, 1] = [0.5, -0.25, 0.0]
    MapOptimizer(m, cfg).step(g)
    step = host(m, "color")[0, 1] - before[0, 1]
    assert step[0] == pytest.approx(-cfg.lr_color, rel=1e-6)
    assert step[1] == pytest.approx(cfg.lr_color, rel=1e-6)
    assert step[2] == 0.0
    np.testing.assert_array_equal(host(m, "color")[0, 0], before[0, 0])


def test_zero_gradients_leave_the_map_unchanged():
    m, _, _ = three_gaussians(np.random.default_rng(1))
    names = ("color", "log_radius", "opacity_logit", "delta")
    snap = {k: host(m, k) for k in names}
    MapOptimizer(m, MapperConfig()).step(zero_grads(m))
    for k in names:
        np.testing.assert_array_equal(host(m, k), snap[k])


def test_frozen_offset_is_not_updated():
    m, _, _ = three_gaussians(np.random.default_rng(2))
    delta = host(m, "delta")
    g = zero_grads(m)
    g.delta[:] = 1.0
    g.opacity_logit[:] = 1.0
    MapOptimizer(m, MapperConfig(offset_frozen=True)).step(g)
    np.testing.assert_array_equal(host(m, "delta"), delta)
    assert np.any(host(m, "opacity_logit") != 0.0)


def test_colours_clipped_to_unit_range():
    m, _, _ = three_gaussians(np.random.default_rng(3))
    m.color[:] = 0.001
    g = zero_grads(m)
    g.color[:] = 1.0
    MapOptimizer(m, MapperConfig(lr_color=0.01)).step(g)
    assert host(m, "color").min() >= 0.0


def test_radius_gradient_chained_through_log_radius():
    m, _, _ = three_gaussians(np.random.default_rng(4))
    logr = host(m, "log_radius")
    g = zero_grads(m)
    g.radius[0, 2] = 0.7
    MapOptimizer(m, MapperConfig()).step(g)
    moved = host(m, "log_radius") != logr
    assert moved[0, 2] and moved.sum() == 1
    assert host(m, "log_radius")[0, 2] < logr[0, 2]  # sign(g_radius * radius), radius > 0


def rendered_target(maps, pose, intr):
    out = splat(maps, pose, intr)
    depth = np_(out.depth).astype(np.float32)
    return SimpleNamespace(color=np.clip(np_(out.color), 0.0, 1.0).astype(np.float32),
                           depth=depth, valid_mask=np.ones(depth.shape, dtype=bool),
                           intrinsics=intr, index=0)


def test_perfect_target_zero_loss_and_smooth_gradients():
    m, pose, intr = three_gaussians(np.random.default_rng(10))
    frame = rendered_target([m], pose, intr)
    bd, _, _ = mapping_loss([m], frame, pose, MapperConfig())
    assert bd.total < 1e-6
    # SSIM only: the L1 terms' signs at fp32 quantisation are +-1, not 0
    _, g, _ = mapping_loss([m], frame, pose, MapperConfig(rho=0.0, tau=1.0, sigma=0.0))
    for x in (g.color, g.radius, g.opacity_logit, g.delta):
        assert np.abs(np_(x)).max() < 1e-6


def test_breakdown_composition_with_masked_depth():
    m, pose, intr = three_gaussians(np.random.default_rng(11))
    frame = rendered_target([m], pose, intr)
    frame.color[:] = np.clip(frame.color + 0.1, 0.0, 1.0)
    frame.depth[:] += 0.05
    frame.valid_mask[:, : intr.width // 2] = False
    bd, _, out = mapping_loss([m], frame, pose, MapperConfig(rho=0.7, tau=0.2, sigma=1.5))
    c = np.abs(np_(out.color) - frame.color.astype(np.float64)).mean()
    d = np.abs(np_(out.depth) - frame.depth.astype(np.float64))[frame.valid_mask].mean()
    assert bd.color_l1 == pytest.approx(c, rel=1e-9)
    assert bd.depth_l1 == pytest.approx(d, rel=1e-9)
    assert bd.total == pytest.approx(0.7 * c + 0.2 * bd.ssim_term + 1.5 * d, rel=1e-9)


def test_frame_without_valid_depth_is_finite():
    m, pose, intr = three_gaussians(np.random.default_rng(12))
    frame = rendered_target([m], pose, intr)
    frame.valid_mask[:] = False
    bd, g, _ = mapping_loss([m], frame, pose, MapperConfig())
    assert bd.depth_l1 == 0.0 and np.isfinite(bd.total)
    assert np.all(np.isfinite(np_(g.delta)))


@pytest.mark.parametrize("normalize", [False, True])
def test_assembled_gradient_matches_central_differences(normalize):
    rng = np.random.default_rng(13 + normalize)
    cfg = MapperConfig(normalize_depth=normalize)
    checked = 0
    for _ in range(2000):
        if checked == 3:
            break
        m, pose, intr = three_gaussians(rng)
        if not fd_safe(m, pose, intr, margin=0.01):
            continue
        h, w = intr.height, intr.width
        frame = SimpleNamespace(color=rng.uniform(0.1, 0.9, (h, w, 3)).astype(np.float32),
                                depth=rng.uniform(0.7, 1.3, (h, w)).astype(np.float32),
                                valid_mask=np.ones((h, w), dtype=bool), intrinsics=intr, index=0)
        _, g, _ = mapping_loss([m], frame, pose, cfg)
        radius = np_(m.radius)
        analytic = {2: np_(g.radius) * radius, 3: np_(g.opacity_logit), 1: np_(g.delta)}
        gcol = np_(g.color)
        P = m.planes  # [7, 1, 3]
        for plane in (1, 2, 3, 4, 5, 6):
            for k in rng.choice(3, size=3, replace=False):
                orig = float(P[plane, 0, k])
                step = 1e-5 * max(1.0, abs(orig))
                P[plane, 0, k] = orig + step
                lp = mapping_loss([m], frame, pose, cfg, with_grads=False)[0].total
                P[plane, 0, k] = orig - step
                lm = mapping_loss([m], frame, pose, cfg, with_grads=False)[0].total
                P[plane, 0, k] = orig
                fd = (lp - lm) / (2 * step)
                ana = gcol[0, k, plane - 4] if plane >= 4 else analytic[plane][0, k]
                assert abs(fd - ana) / max(abs(fd), abs(ana), 1e-6) < 2e-3, (plane, k, fd, ana)
        checked += 1
    assert checked == 3
