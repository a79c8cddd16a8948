"""Pin the oracle's render-based pose initialiser (oracle/track.py,
restating tracker.py:354-426) against the reference's own result on the C1
scene (tests/golden/render_init.npz).  No GPU needed."""

from types import SimpleNamespace

import numpy as np
import pytest

from oracle import track as OT
from paper_2603_21055_b200 import scenes
from paper_2603_21055_b200.geometry import Pose


def _case():
    intr, fa, fb, params, truth = scenes.config_render_init()
    m = SimpleNamespace(frame_index=0, pose=Pose.identity(), intrinsics=intr,
                        base_depth=params.base_depth, delta=params.delta,
                        log_radius=params.log_radius, opacity_logit=params.opacity_logit,
                        color=params.color, active_mask=params.active_mask)
    return intr, fb, m


@pytest.mark.parametrize("iters", [1, 10])
def test_render_init_matches_reference(golden, iters):
    g = golden("render_init")
    intr, fb, m = _case()
    rot, t, ok = OT.init_pose_render(fb.color, fb.depth, fb.valid_mask, m, np.eye(3),
                                     np.zeros(3), intr, iters=iters)
    assert ok == bool(g[f"it{iters}_ok"])
    np.testing.assert_allclose(rot, g[f"it{iters}_R"], atol=1e-9)
    np.testing.assert_allclose(t, g[f"it{iters}_t"], atol=1e-9)


def test_render_init_low_coverage(golden):
    g = golden("render_init")
    intr, fb, m = _case()
    rot, t, ok = OT.init_pose_render(fb.color, fb.depth, fb.valid_mask, m, np.eye(3),
                                     np.array([5.0, 0.0, 0.0]), intr, iters=3)
    assert not ok and not bool(g["far_ok"])
    np.testing.assert_array_equal(t, g["far_t"])
