"""The CPU oracle pinned at the benchmark's own configurations: one view of
the C3 and C4 windows (init_params and the teacher-forced state) against the
reference-run fixtures tests/golden/bench_*.npz (make_golden.py
golden_bench).  The GPU path is held to the same fixtures in
tests/test_bench_parity_gpu.py; this pins the checker itself there."""

import os
from types import SimpleNamespace

import numpy as np
import pytest

from helpers import forced_params, rel_err, tile_digest
from oracle import raster as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


# (C4's teacher-forced view is checked on the GPU only: ~50 s of CPU here)
@pytest.mark.parametrize("cfg,state", [("c3", "init"), ("c3", "forced"), ("c4", "init")])
def test_oracle_vs_reference_bench_view(cfg, state):
    from paper_2603_21055_b200 import scenes
    g = dict(np.load(os.path.join(GOLDEN, f"bench_{cfg}_{state}.npz")))
    wc = scenes.config_c3() if cfg == "c3" else scenes.config_c4()
    params = wc.params if state == "init" else forced_params(wc.params)
    v = int(g["view"])
    maps = [SimpleNamespace(frame_index=i, pose=wc.poses[i], intrinsics=wc.intr,
                            base_depth=p.base_depth, delta=p.delta, log_radius=p.log_radius,
                            opacity_logit=p.opacity_logit, color=p.color,
                            active_mask=p.active_mask) for i, p in enumerate(params)]
    pose = wc.poses[v]
    b = O.prepare(maps, pose.rotation, pose.translation, wc.intr, learnable="all")
    assert len(b) == int(g["n_surv"])
    off, lst = O.tile_lists(b)
    np.testing.assert_array_equal(off, g["offsets"])
    got = tile_digest(off, b.frame[lst], b.pixel_index[lst])
    assert np.array_equal(got, g["tile_hash"]), int((got != g["tile_hash"]).sum())
    fr = wc.frames[v]
    loss, grads, out = O.mapping_loss(maps, fr.color, fr.depth, fr.valid_mask, pose.rotation,
                                      pose.translation, wc.intr, learnable_map="all")
    np.testing.assert_allclose([loss.color_l1, loss.depth_l1], g["loss"], rtol=1e-12)
    px = g["px"]
    np.testing.assert_allclose(out.color.reshape(-1, 3)[px], g["px_color"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(out.depth.reshape(-1)[px], g["px_depth"], rtol=0, atol=1e-12)
    np.testing.assert_array_equal(out.contributors.reshape(-1)[px], g["px_count"])
    planes = [np.stack([m.delta, m.radius, m.opacity_logit, *np.moveaxis(m.color, 2, 0)])
              for m in grads]
    flat = np.concatenate([p.reshape(6, -1).T for p in planes])[g["gs"]]
    for c in range(6):
        assert rel_err(flat[:, c], g["g_sample"][:, c], floor_frac=1e-6) < 1e-9, c
    sums = np.stack([p.reshape(6, -1).sum(axis=1) for p in planes])
    assert float((np.abs(sums - g["g_frame_sums"]) /
                  np.maximum(g["g_frame_abs"], 1e-300)).max()) < 1e-9
