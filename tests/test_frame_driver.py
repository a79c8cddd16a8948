"""The per-frame mapping driver and its formats against
the reference's own outputs (tests/golden/frame_driver.npz):
target_schedule (mapper.py:175-194), inpaint_depth (datasets.py:368-398),
assemble_base_depth (:197-214), map_frame (:217-247) and the .bin map file
(gaussians.py:118-180)."""

import os

import numpy as np
import pytest

from oracle import track as OT


def _intr():
    from paper_2603_21055_b200 import scenes
    return scenes.config_render_init()[0]


def test_target_schedule_matches_reference(golden):
    from paper_2603_21055_b200.mapper import target_schedule
    g = golden("frame_driver")
    i = 0
    while f"sched{i}" in g:
        it, n, frac, seed = g[f"sched{i}_args"]
        got = target_schedule(int(it), int(n), float(frac), int(seed))
        np.testing.assert_array_equal(got, g[f"sched{i}"])
        i += 1


def test_oracle_inpaint_matches_reference(golden):
    g = golden("frame_driver")
    np.testing.assert_array_equal(OT.inpaint_depth(g["inpaint_in"], g["inpaint_valid"]),
                                  g["inpaint_out"])
    np.testing.assert_array_equal(OT.inpaint_depth(g["inpaint_in"], g["inpaint_valid"],
                                                   max_iters=7), g["inpaint_out_short"])


def test_map_file_bytes_and_load_cpu(golden, tmp_path):
    """Writer and reader on CPU tensors: byte-identical to the reference's file."""
    from paper_2603_21055_b200.gaussians import (GaussianMapError, PixelGaussianMap,
                                                 load_gaussian_map, save_gaussian_map)
    from paper_2603_21055_b200.geometry import Pose
    g = golden("frame_driver")
    blob = g["mapfile"].tobytes()
    ref = tmp_path / "ref.bin"
    ref.write_bytes(blob)
    intr = _intr()
    m = load_gaussian_map(ref, intr, device="cpu")
    out = tmp_path / "ours.bin"
    save_gaussian_map(out, m)
    assert out.read_bytes() == blob
    assert m.frame_index == 1 and m.shape == g["mf_base_depth"].shape
    np.testing.assert_array_equal(m.active_mask.numpy(), g["mf_active_mask"])
    np.testing.assert_array_equal(m.base_depth.numpy(),
                                  g["mf_base_depth"].astype(np.float32).astype(np.float64))
    bad = tmp_path / "bad.bin"
    bad.write_bytes(blob[:-1])
    with pytest.raises(GaussianMapError, match="bad.bin"):
        load_gaussian_map(bad, intr, device="cpu")
    bad.write_bytes(b"XXXX" + blob[4:])
    with pytest.raises(GaussianMapError, match="magic"):
        load_gaussian_map(bad, intr, device="cpu")


@pytest.mark.gpu
def test_gpu_inpaint_bit_exact(golden):
    from paper_2603_21055_b200.depthfill import inpaint_depth
    g = golden("frame_driver")
    out, sweeps = inpaint_depth(g["inpaint_in"], g["inpaint_valid"], return_sweeps=True)
    np.testing.assert_array_equal(out, g["inpaint_out"])
    assert 0 < sweeps <= 200
    np.testing.assert_array_equal(inpaint_depth(g["inpaint_in"], g["inpaint_valid"], max_iters=7),
                                  g["inpaint_out_short"])
    # fully valid input: unchanged (idempotent)
    full = np.where(g["inpaint_valid"], g["inpaint_in"], 1.0)
    np.testing.assert_array_equal(inpaint_depth(full, full > 0), full)


def _gpu_case():
    import torch
    from paper_2603_21055_b200 import scenes
    from paper_2603_21055_b200.gaussians import PixelGaussianMap
    from paper_2603_21055_b200.geometry import Pose
    from paper_2603_21055_b200.scenes import Frame
    intr, fa, fb, params, truth = scenes.config_render_init()
    map_a = PixelGaussianMap(0, Pose.identity(), intr, params.base_depth, params.delta,
                             params.color, params.log_radius, params.opacity_logit,
                             params.active_mask, dtype=torch.float64)
    return intr, fa, fb, map_a, truth


@pytest.mark.gpu
def test_gpu_assemble_base_depth(golden):
    from paper_2603_21055_b200.mapper import assemble_base_depth
    from paper_2603_21055_b200.scenes import Frame
    g = golden("frame_driver")
    intr, fa, fb, map_a, truth = _gpu_case()
    fr = Frame(fb.color, g["target_depth"], g["target_valid"], intr, index=1)
    base = assemble_base_depth(fr, truth, [map_a])
    np.testing.assert_allclose(base, g["base_depth"], rtol=0, atol=1e-9)


@pytest.mark.gpu
def test_gpu_map_frame(golden):
    """map_frame on the GPU vs the oracle replay of the same loop and vs the
    reference's own run.  The first render is the fresh map seen from its own
    view, where every neighbour Gaussian at 3 px sits exactly on the 3-sigma
    boundary (d2 = 9 s2 in real arithmetic; sigma = exp(log(D/fx)) fx/D) and
    the inclusion is decided by the last ulp of exp and of the base depth --
    the reference's own answer depends on the host's numpy SIMD exp path
    (D7).  The knife-edge pixels then move the loss by ~1e-4
    relative, so the loop is checked at that level here; its pieces are
    checked tightly elsewhere (schedule exact, base depth 1e-9, loss /
    gradients / Adam at 1e-9 in the C1 and tau tests)."""
    from oracle import raster as O
    from paper_2603_21055_b200.geometry import Pose
    from paper_2603_21055_b200.mapper import MapperConfig, map_frame
    from paper_2603_21055_b200.scenes import Frame
    g = golden("frame_driver")
    intr, fa, fb, map_a, truth = _gpu_case()
    fr_b = Frame(fb.color, g["target_depth"], g["target_valid"], intr, index=1)
    fr_a = Frame(fa.color, fa.depth, fa.valid_mask, intr, index=0)
    gmap, losses = map_frame(fr_b, truth, [(fr_a, Pose.identity(), map_a)],
                             MapperConfig(mapping_iters=4), seed=0)
    om, olosses = O.map_frame(fb.color, g["target_depth"], g["target_valid"], truth.rotation,
                              truth.translation, 1, intr, gmap.base_depth.cpu().numpy(),
                              [(fa.color, fa.depth, fa.valid_mask, np.eye(3), np.zeros(3),
                                map_a.to_numpy())], 4)
    # vs the oracle replay (same fp64 exp, same knife-edge decisions): tight
    np.testing.assert_allclose(losses, olosses, rtol=1e-10)
    for k in ("delta", "log_radius", "opacity_logit", "color"):
        d = np.abs(getattr(gmap, k).cpu().numpy() - getattr(om, k))
        assert d.max() < 1e-9, (k, d.max())
    # vs the reference's own run: the knife-edge inclusions differ (D7), the
    # loss moves by ~1e-4 relative
    np.testing.assert_allclose(losses, g["mf_losses"], rtol=1e-3)
    np.testing.assert_array_equal(gmap.active_mask.cpu().numpy(), g["mf_active_mask"])
    np.testing.assert_allclose(gmap.base_depth.cpu().numpy(), g["mf_base_depth"], atol=1e-9)


@pytest.mark.gpu
def test_gpu_map_frame_deterministic(golden, tmp_path):
    """Run twice, map_frame gives byte-identical maps and map files (the
    reference's pipeline is bit-reproducible across runs and worker counts,
    reference tests/test_pipeline.py:76-85): the exact backward sums in
    integer fixed point, so atomic ordering cannot change a bit."""
    from paper_2603_21055_b200.gaussians import save_gaussian_map
    from paper_2603_21055_b200.geometry import Pose
    from paper_2603_21055_b200.mapper import MapperConfig, map_frame
    from paper_2603_21055_b200.scenes import Frame
    g = golden("frame_driver")
    intr, fa, fb, map_a, truth = _gpu_case()
    fr_b = Frame(fb.color, g["target_depth"], g["target_valid"], intr, index=1)
    fr_a = Frame(fa.color, fa.depth, fa.valid_mask, intr, index=0)
    outs = []
    for k in range(2):
        gmap, losses = map_frame(fr_b, truth, [(fr_a, Pose.identity(), map_a)],
                                 MapperConfig(mapping_iters=6), seed=0)
        path = tmp_path / f"m{k}.bin"
        save_gaussian_map(str(path), gmap)
        outs.append((gmap.planes.cpu().numpy().tobytes(), path.read_bytes(), losses))
    assert outs[0][0] == outs[1][0]
    assert outs[0][1] == outs[1][1]
    # (the reported losses add per-warp partial sums with fp64 atomics: an
    # ulp apart run to run; they do not feed the update)
    np.testing.assert_allclose(outs[0][2], outs[1][2], rtol=1e-12)
