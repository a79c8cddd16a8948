"""GPU render-based pose initialiser (tracker.init_pose_render) vs the
reference's own result (tests/golden/render_init.npz, tracker.py:354-426).
Bar (north_star): pose within 1e-5 rad / m after the same iterations."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _case():
    from paper_2603_21055_b200 import scenes
    from paper_2603_21055_b200.gaussians import PixelGaussianMap
    from paper_2603_21055_b200.geometry import Pose
    intr, fa, fb, p, truth = scenes.config_render_init()
    m = PixelGaussianMap(0, Pose.identity(), intr, p.base_depth, p.delta, p.color, p.log_radius,
                         p.opacity_logit, p.active_mask, dtype=torch.float64)
    return fb, m


@pytest.mark.parametrize("iters", [1, 10])
def test_render_init_matches_reference(golden, iters):
    from paper_2603_21055_b200.geometry import Pose, pose_difference
    from paper_2603_21055_b200.tracker import init_pose_render
    g = golden("render_init")
    fb, m = _case()
    pose, ok = init_pose_render(fb, m, Pose.identity(), iters=iters)
    assert ok == bool(g[f"it{iters}_ok"])
    rot_err, t_err = pose_difference(pose, Pose(g[f"it{iters}_R"], g[f"it{iters}_t"]))
    assert rot_err < 1e-5 and t_err < 1e-5, (rot_err, t_err)
    np.testing.assert_allclose(pose.translation, g[f"it{iters}_t"], atol=1e-9)


def test_render_init_low_coverage(golden):
    from paper_2603_21055_b200.geometry import Pose
    from paper_2603_21055_b200.tracker import init_pose_render
    fb, m = _case()
    far = Pose(np.eye(3), np.array([5.0, 0.0, 0.0]))
    pose, ok = init_pose_render(fb, m, far, iters=3)
    assert not ok and pose is far
