"""The reference's tracking known-answer tests (raysplat tests/test_tracker.py
TestBuildLocalSet :41-115, TestGlobalSet :117-168, TestGicp :199-320),
restated against the GPU tracker.  Local sets come from depth images through
the 5x5 window fit (delta D2) instead of K-NN over a point cloud, so the
point-cloud GICP draws are replaced by depth frames of a seeded scene seen
from a known pose; the properties checked are the reference's."""

from types import SimpleNamespace

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2603_21055_b200 import scenes
from paper_2603_21055_b200.geometry import Intrinsics, Pose, pose_difference, se3_exp
from paper_2603_21055_b200.tracker import (GlobalGeomSet, LocalGeomSet, TrackerConfig,
                                           TrackerError, build_local_set, gicp_align,
                                           update_global_set)


def flat_frame(depth=2.0, w=64, h=48, fx=100.0):
    intr = Intrinsics(fx=fx, fy=fx, cx=(w - 1) / 2, cy=(h - 1) / 2, width=w, height=h)
    return SimpleNamespace(color=np.full((h, w, 3), 0.5, np.float32),
                           depth=np.full((h, w), depth, np.float32),
                           valid_mask=np.ones((h, w), bool), intrinsics=intr, index=0)


def scene_frame(pose=None, w=160, h=120):
    intr = Intrinsics(fx=120.0, fy=120.0, cx=(w - 1) / 2, cy=(h - 1) / 2, width=w, height=h)
    return scenes.render_frame(scenes.corner_spheres_scene(0), pose or Pose.identity(), intr)


def n(x):
    return x.detach().cpu().numpy() if torch.is_tensor(x) else np.asarray(x)


# ------------------------------------------------------------------ local sets

def test_plane_normals_face_the_camera():
    local = build_local_set(flat_frame(), TrackerConfig(downsample_ratio=4))
    np.testing.assert_allclose(n(local.normals), [[0.0, 0.0, -1.0]] * len(local), atol=1e-4)


def test_vga_grid_count():
    local = build_local_set(flat_frame(w=640, h=480, fx=525.0), TrackerConfig(downsample_ratio=10))
    assert len(local) == 64 * 48


def test_count_follows_the_sample_grid():
    local = build_local_set(flat_frame(w=50, h=30), TrackerConfig(downsample_ratio=7))
    assert len(local) == int(np.ceil(50 / 7)) * int(np.ceil(30 / 7))


def test_ellipse_scales_have_unit_norm():
    local = build_local_set(scene_frame(), TrackerConfig(downsample_ratio=5, scale_mode="ellipse"))
    np.testing.assert_allclose(np.linalg.norm(n(local.scales), axis=1), 1.0, atol=1e-9)


def test_plane_mode_scales_are_fixed():
    local = build_local_set(scene_frame(), TrackerConfig(downsample_ratio=5, scale_mode="plane"))
    np.testing.assert_allclose(n(local.scales), [[1.0, 1.0, 1e-3]] * len(local))


def test_none_mode_keeps_metric_scales():
    s = n(build_local_set(flat_frame(), TrackerConfig(downsample_ratio=4, scale_mode="none")).scales)
    assert s[:, 0].max() < 0.1
    assert np.all(s[:, 2] <= s[:, 0] * 2e-3)
    assert np.all(s > 0)


def test_rotations_orthonormal_with_the_normal_as_third_column():
    local = build_local_set(scene_frame(), TrackerConfig(downsample_ratio=6))
    r = n(local.rotations)
    eye = np.einsum("nij,nkj->nik", r, r)
    np.testing.assert_allclose(eye, np.broadcast_to(np.eye(3), eye.shape), atol=1e-9)
    np.testing.assert_allclose(np.linalg.det(r), 1.0, atol=1e-9)
    np.testing.assert_allclose(r[:, :, 2], n(local.normals), atol=1e-12)


def test_too_few_valid_pixels_raise():
    f = flat_frame(w=16, h=16)
    f.valid_mask[:] = False
    f.valid_mask[0, :3] = True
    with pytest.raises(TrackerError, match="valid pixels"):
        build_local_set(f, TrackerConfig())


def test_collinear_neighbourhoods_are_floored_not_nan():
    f = flat_frame()
    f.valid_mask[:] = False
    f.valid_mask[8, :] = True  # one sampled row: collinear back-projections
    s = n(build_local_set(f, TrackerConfig(downsample_ratio=4)).scales)
    assert np.all(np.isfinite(s)) and np.all(s > 0)


@pytest.mark.parametrize("kw", [dict(downsample_ratio=0), dict(neighbor_count=3),
                                dict(scale_mode="banana"), dict(metric_mode="euclid"),
                                dict(init_mode="warp")])
def test_config_validation(kw):
    with pytest.raises(TrackerError):
        TrackerConfig(**kw)


# ------------------------------------------------------------------ global set

def points_set(pts):
    m = len(pts)
    return LocalGeomSet(pts, np.broadcast_to(np.eye(3), (m, 3, 3)).copy(),
                        np.full((m, 3), 1 / np.sqrt(3)), np.tile([0.0, 0.0, 1.0], (m, 1)))


def test_first_insert_of_distinct_cells_adds_all():
    g = GlobalGeomSet(voxel_size=0.001)
    pts = np.random.default_rng(0).uniform(0, 1, (200, 3))
    assert update_global_set(g, points_set(pts), Pose.identity()) == 200 and len(g) == 200


def test_reinserting_adds_nothing():
    f = scene_frame()
    local = build_local_set(f, TrackerConfig(downsample_ratio=8))
    g = GlobalGeomSet(voxel_size=0.02)
    first = update_global_set(g, local, Pose.identity())
    assert first > 0
    assert update_global_set(g, local, Pose.identity()) == 0 and len(g) == first


def test_one_member_per_voxel():
    g = GlobalGeomSet(voxel_size=0.05)
    update_global_set(g, points_set(np.random.default_rng(1).uniform(0, 0.1, (300, 3))),
                      Pose.identity())
    cells = {tuple(k) for k in np.floor(n(g.centers) / 0.05).astype(np.int64)}
    assert len(cells) == len(g)


def test_disjoint_clouds_add_up():
    rng = np.random.default_rng(2)
    g = GlobalGeomSet(voxel_size=0.001)
    na = update_global_set(g, points_set(rng.uniform(0, 1, (150, 3))), Pose.identity())
    nb = update_global_set(g, points_set(rng.uniform(10, 11, (150, 3))), Pose.identity())
    assert len(g) == na + nb == 300


def test_world_transform_applied_on_insert():
    local = build_local_set(scene_frame(), TrackerConfig(downsample_ratio=6))
    pose = se3_exp([0.1, -0.2, 0.05, 0.3, 0.1, -0.2])
    g = GlobalGeomSet(voxel_size=1e-4)
    assert update_global_set(g, local, pose) == len(local)
    np.testing.assert_allclose(n(g.centers), pose.apply(n(local.centers)), atol=1e-12)
    np.testing.assert_allclose(n(g.normals), n(local.normals) @ pose.rotation.T, atol=1e-12)
    np.testing.assert_allclose(np.linalg.det(n(g.rotations)), 1.0, atol=1e-9)


def test_querying_an_empty_set_raises():
    with pytest.raises(TrackerError, match="empty"):
        GlobalGeomSet().query_nearest(np.zeros((1, 3)))


# ------------------------------------------------------------------ GICP

def frame_pair(seed, twist_scale=1.0):
    """Global set from the scene seen at identity (fine voxels); the local set
    is the frame rendered from a known offset pose."""
    rng = np.random.default_rng(seed)
    true = se3_exp(twist_scale * np.concatenate([rng.uniform(-0.03, 0.03, 3),
                                                 rng.uniform(-0.05, 0.05, 3)]))
    g = GlobalGeomSet(voxel_size=1e-4)
    update_global_set(g, build_local_set(scene_frame(), TrackerConfig(downsample_ratio=1)),
                      Pose.identity())
    local = build_local_set(scene_frame(true), TrackerConfig(downsample_ratio=2))
    return local, g, true


def test_true_pose_is_a_fixed_point():
    local, g, true = frame_pair(3)
    pose, diag = gicp_align(local, g, true, TrackerConfig())
    dr, dt = pose_difference(pose, true)
    assert not diag.failed and dr < 1e-3 and dt < 1e-3


@pytest.mark.parametrize("seed", [4, 5])
def test_known_transform_recovered_from_identity(seed):
    local, g, true = frame_pair(seed)
    pose, diag = gicp_align(local, g, Pose.identity(), TrackerConfig(max_gicp_iters=40))
    dr, dt = pose_difference(pose, true)
    assert not diag.failed and dr < np.deg2rad(0.2) and dt < 5e-3


def test_cost_does_not_increase_across_accepted_steps():
    local, g, _ = frame_pair(6)
    _, diag = gicp_align(local, g, Pose.identity(), TrackerConfig())
    assert diag.cost_pairs
    for before, after in diag.cost_pairs:
        assert after <= before + 1e-12


def test_too_few_inliers_returns_the_initial_pose_flagged():
    local, g, _ = frame_pair(7)
    init = Pose(np.eye(3), np.array([50.0, 50.0, 50.0]))  # off every surface
    pose, diag = gicp_align(local, g, init, TrackerConfig())
    assert diag.failed and np.array_equal(pose.translation, init.translation)


# ------------------------------------------------------------------ 3x3 eig (T3)
# raysplat tests/test_geometry.py TestSym3Eig :186-244 on sym_eigh3_batch

def eig(mats):
    from paper_2603_21055_b200.tracker import sym_eigh3_batch
    rot, vals = sym_eigh3_batch(np.asarray(mats, dtype=np.float64).reshape(-1, 3, 3))
    return n(rot), n(vals)


def test_eig_known_diagonal():
    r, v = eig(np.diag([4.0, 1.0, 0.25]))
    np.testing.assert_allclose(v[0], [4.0, 1.0, 0.25], atol=1e-12)
    np.testing.assert_allclose(np.abs(r[0]), np.eye(3), atol=1e-12)


def test_eig_identity():
    r, v = eig(np.eye(3))
    np.testing.assert_allclose(v[0], np.ones(3), atol=1e-12)
    np.testing.assert_allclose(r[0] @ r[0].T, np.eye(3), atol=1e-12)


def test_eig_random_spd_reconstruction():
    rng = np.random.default_rng(31)
    a = rng.normal(size=(500, 3, 3))
    m = a @ a.transpose(0, 2, 1) + 1e-6 * np.eye(3)
    r, v = eig(m)
    recon = np.einsum("nij,nj,nkj->nik", r, v, r)
    assert np.linalg.norm(recon - m, axis=(1, 2)).max() < 1e-7
    np.testing.assert_allclose(np.einsum("nij,nkj->nik", r, r),
                               np.broadcast_to(np.eye(3), (500, 3, 3)), atol=1e-9)
    assert (np.linalg.det(r) > 0).all()
    assert (v[:, 0] >= v[:, 1]).all() and (v[:, 1] >= v[:, 2]).all()


def test_eig_rank_deficient():
    r, v = eig(np.diag([2.0, 1.0, 0.0]))
    np.testing.assert_allclose(v[0], [2.0, 1.0, 0.0], atol=1e-12)
    np.testing.assert_allclose(np.abs(r[0][:, 2]), [0.0, 0.0, 1.0], atol=1e-12)


def test_eig_near_degenerate_pair():
    m = np.diag([1.0, 1.0 + 1e-13, 2.0])
    r, v = eig(m)
    recon = r[0] @ np.diag(v[0]) @ r[0].T
    assert np.linalg.norm(recon - m) < 1e-7
