"""The reference's per-frame mapping KATs (raysplat tests/test_mapper.py
TestSchedule :29-57 on the host, TestMapFrame :238-322 on the GPU):
the target schedule's floor and round-robin, map_frame's convergence,
determinism, frozen neighbours, hole filling from a neighbour render or by
inpainting, the no-valid-depth error, and mapping_step's loss breakdown.
The frame is a seeded room corner (checkered floor and walls, three
spheres) rendered with this repo's ray caster."""

from types import SimpleNamespace

import numpy as np
import pytest

from paper_2603_21055_b200.geometry import Intrinsics, Pose
from paper_2603_21055_b200.mapper import target_schedule


def test_schedule_without_neighbours_is_all_current():
    assert target_schedule(7, 0, 0.4) == [0] * 7


def test_schedule_floor_ten_iterations_one_neighbour():
    s = target_schedule(10, 1, 0.4)
    assert s.count(0) >= 4 and set(s) == {0, 1}


def test_schedule_prefix_floor_and_round_robin():
    for iters, nn, frac in [(10, 1, 0.4), (100, 3, 0.4), (50, 2, 0.5), (33, 5, 0.25)]:
        s = target_schedule(iters, nn, frac)
        cur = 0
        for i, slot in enumerate(s):
            assert 0 <= slot <= nn
            cur += slot == 0
            assert cur >= frac * (i + 1) - 1e-12
        for j, x in enumerate([x for x in s if x != 0]):
            assert x == 1 + j % nn


def test_schedule_deterministic_and_seed_rotates_neighbours():
    a = target_schedule(20, 3, 0.4, seed=5)
    assert a == target_schedule(20, 3, 0.4, seed=5)
    b = target_schedule(20, 3, 0.4, seed=6)
    na, nb = [x for x in a if x != 0], [x for x in b if x != 0]
    assert nb[0] == 1 + (na[0] % 3)


# ------------------------------------------------------------------ GPU

INTR = Intrinsics(fx=80.0, fy=80.0, cx=63.5, cy=47.5, width=128, height=96)


def room_frame():
    """Checkered floor and walls with three spheres, 1-3 m away."""
    from paper_2603_21055_b200 import scenes
    return scenes.render_frame(scenes.corner_spheres_scene(0), Pose.identity(), INTR, 0,
                               device="cuda"), Pose.identity()


def np_(x):
    return x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)


@pytest.mark.gpu
def test_map_frame_converges_on_a_textured_frame():
    from paper_2603_21055_b200.mapper import MapperConfig, map_frame
    from paper_2603_21055_b200.rasterizer import splat
    frame, pose = room_frame()
    gmap, losses = map_frame(frame, pose, [], MapperConfig(mapping_iters=60))
    assert len(losses) == 60
    assert losses[-1] < 0.3 * losses[0]
    assert np.median(losses[40:]) < np.median(losses[:10])
    out = np_(splat([gmap], pose, INTR).color)
    mse = float(np.mean((out - frame.color.astype(np.float64)) ** 2))
    assert 10.0 * np.log10(1.0 / mse) > 28.0


@pytest.mark.gpu
def test_map_frame_is_deterministic():
    from paper_2603_21055_b200.mapper import MapperConfig, map_frame
    frame, pose = room_frame()
    cfg = MapperConfig(mapping_iters=8)
    a, la = map_frame(frame, pose, [], cfg, seed=3)
    b, lb = map_frame(frame, pose, [], cfg, seed=3)
    np.testing.assert_allclose(la, lb, rtol=1e-12)  # (fp64 loss sums are atomics)
    for k in ("color", "delta", "log_radius"):
        np.testing.assert_allclose(np_(getattr(a, k)), np_(getattr(b, k)), rtol=0, atol=1e-12)


@pytest.mark.gpu
def test_neighbour_map_is_never_updated():
    from paper_2603_21055_b200.gaussians import init_gaussians
    from paper_2603_21055_b200.mapper import MapperConfig, map_frame
    frame, pose = room_frame()
    nmap = init_gaussians(frame, pose)
    nmap.opacity_logit[:] = 1.0
    snap = np_(nmap.planes).copy()
    map_frame(frame, pose, [(frame, pose, nmap)], MapperConfig(mapping_iters=6))
    np.testing.assert_array_equal(np_(nmap.planes), snap)


@pytest.mark.gpu
def test_hole_filled_from_a_neighbour_render():
    from paper_2603_21055_b200.gaussians import init_gaussians
    from paper_2603_21055_b200.mapper import assemble_base_depth
    frame, pose = room_frame()
    nmap = init_gaussians(frame, pose)
    nmap.opacity_logit[:] = 2.0
    depth, mask = frame.depth.copy(), frame.valid_mask.copy()
    depth[30:38, 40:48] = 0.0
    mask[30:38, 40:48] = False
    holed = SimpleNamespace(color=frame.color, depth=depth, valid_mask=mask, intrinsics=INTR,
                            timestamp=0.0, index=1)
    base = assemble_base_depth(holed, pose, [nmap])
    patch = base[30:38, 40:48]
    assert np.all(patch > 0)
    assert np.abs(patch - frame.depth[30:38, 40:48].astype(np.float64)).max() < 0.05
    np.testing.assert_array_equal(base[mask], frame.depth[mask].astype(np.float64))


@pytest.mark.gpu
def test_hole_without_neighbour_is_inpainted():
    from paper_2603_21055_b200.mapper import assemble_base_depth
    frame, pose = room_frame()
    depth, mask = frame.depth.copy(), frame.valid_mask.copy()
    depth[10:14, 10:14] = 0.0
    mask[10:14, 10:14] = False
    holed = SimpleNamespace(color=frame.color, depth=depth, valid_mask=mask, intrinsics=INTR,
                            timestamp=0.0, index=1)
    assert np.all(assemble_base_depth(holed, pose, []) > 0)


@pytest.mark.gpu
def test_frame_without_valid_depth_raises():
    from paper_2603_21055_b200.mapper import MapperConfig, map_frame
    frame, pose = room_frame()
    dead = SimpleNamespace(color=frame.color, depth=np.zeros_like(frame.depth),
                           valid_mask=np.zeros_like(frame.valid_mask), intrinsics=INTR,
                           timestamp=0.0, index=2)
    with pytest.raises(ValueError, match="no valid depth"):
        map_frame(dead, pose, [], MapperConfig(mapping_iters=2))


@pytest.mark.gpu
def test_mapping_step_reports_its_loss():
    from paper_2603_21055_b200.gaussians import init_gaussians
    from paper_2603_21055_b200.mapper import MapOptimizer, MapperConfig, mapping_step
    frame, pose = room_frame()
    gmap = init_gaussians(frame, pose)
    b = mapping_step(gmap, MapOptimizer(gmap, MapperConfig()), frame, pose, [], MapperConfig())
    assert b.total > 0.0
    assert b.total == pytest.approx(0.8 * b.color_l1 + 0.2 * b.ssim_term + b.depth_l1, rel=1e-12)
