"""The reference's pose-initialiser known-answer tests (raysplat
tests/test_tracker.py TestInitializers :321-349 and TestRenderInit :352-426):
constant-speed extrapolation (host math, CPU) and the render-based
initialiser on the GPU renderer -- a zero-residual fixed point, recovery of
a small shift on a textured and on a textureless scene (the latter through
the depth residual), and the low-coverage fallback.  Scenes are rebuilt from
their descriptions with this repo's ray caster."""

from types import SimpleNamespace

import numpy as np
import pytest

from paper_2603_21055_b200.geometry import Intrinsics, Pose, pose_difference, se3_exp
from paper_2603_21055_b200.tracker import init_pose_constant_speed


def test_constant_speed_zero_velocity():
    p = se3_exp([0.1, 0.2, -0.1, 0.3, 0.0, 1.0])
    dr, dt = pose_difference(init_pose_constant_speed(p, p), p)
    assert dr < 1e-12 and dt < 1e-12


def test_constant_speed_translation():
    q = init_pose_constant_speed(Pose(np.eye(3), np.array([0.01, 0.0, 0.0])), Pose.identity())
    np.testing.assert_allclose(q.translation, [0.02, 0.0, 0.0], atol=1e-15)


def test_constant_speed_rotation():
    step = se3_exp([0.0, 0.0, np.deg2rad(2.0), 0.0, 0.0, 0.0])
    want = se3_exp([0.0, 0.0, np.deg2rad(4.0), 0.0, 0.0, 0.0])
    dr, dt = pose_difference(init_pose_constant_speed(step, Pose.identity()), want)
    assert dr < 1e-12 and dt < 1e-12


# ------------------------------------------------------------------ GPU

INTR = Intrinsics(fx=120.0, fy=120.0, cx=79.5, cy=59.5, width=160, height=120)


def textured_scene():
    """Floor, back and side walls (checkered) and three spheres: a desk-like
    scene that constrains all six degrees of freedom."""
    from paper_2603_21055_b200 import scenes
    return scenes.corner_spheres_scene(0)


def flat_scene():
    """A textureless fronto-parallel wall: only the depth residual constrains
    the motion along the optical axis."""
    from paper_2603_21055_b200 import scenes
    return [scenes.Rect((-4.0, -4.0, 1.5), (8.0, 0.0, 0.0), (0.0, 8.0, 0.0), (0.5, 0.5, 0.5))]


def render(prims, pose, index=0):
    from paper_2603_21055_b200 import scenes
    return scenes.render_frame(prims, pose, INTR, index, device="cuda")


def sharp_map(frame, pose):
    """A near-point-sample map that re-renders the frame almost exactly."""
    from paper_2603_21055_b200.gaussians import init_gaussians
    m = init_gaussians(frame, pose)
    m.opacity_logit[:] = 6.0
    m.log_radius[:] -= np.log(3.0)
    return m


@pytest.mark.gpu
def test_zero_residual_is_a_fixed_point():
    from paper_2603_21055_b200.rasterizer import splat
    from paper_2603_21055_b200.tracker import init_pose_render
    pose = Pose.identity()
    frame = render(textured_scene(), pose)
    m = sharp_map(frame, pose)
    out = splat([m], pose, INTR)
    target = SimpleNamespace(color=np.clip(out.color.cpu().numpy(), 0, 1).astype(np.float32),
                             depth=out.depth.cpu().numpy().astype(np.float32),
                             valid_mask=np.ones(frame.valid_mask.shape, bool), intrinsics=INTR,
                             timestamp=0.0, index=1)
    refined, ok = init_pose_render(target, m, pose, iters=4)
    assert ok
    dr, dt = pose_difference(refined, pose)
    assert dr < 1e-6 and dt < 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("scene,shift", [("textured", [0.0, 0.0, 0.0, 0.01, 0.0, 0.0]),
                                         ("flat", [0.0, 0.0, 0.0, 0.0, 0.0, 0.008])])
def test_recovers_a_small_shift(scene, shift):
    from paper_2603_21055_b200.mapper import MapperConfig, map_frame
    from paper_2603_21055_b200.tracker import init_pose_render
    prims = textured_scene() if scene == "textured" else flat_scene()
    p0 = Pose.identity()
    p1 = se3_exp(shift).compose(p0)
    f0, f1 = render(prims, p0, 0), render(prims, p1, 1)
    m, _ = map_frame(f0, p0, [], MapperConfig(mapping_iters=60))
    refined, ok = init_pose_render(f1, m, p0, iters=10)
    assert ok
    _, dt = pose_difference(refined, p1)
    assert dt < 2e-3


@pytest.mark.gpu
def test_low_coverage_falls_back_to_the_initial_pose():
    from paper_2603_21055_b200.tracker import init_pose_render
    pose = Pose.identity()
    frame = render(textured_scene(), pose)
    m = sharp_map(frame, pose)
    away = se3_exp([0.0, np.pi / 2, 0.0, 0.0, 0.0, 0.0]).compose(pose)
    out, ok = init_pose_render(frame, m, away, iters=3)
    assert not ok
    dr, dt = pose_difference(out, away)
    assert dr == 0.0 and dt == 0.0
