"""GPU parity of the mapping hot path: sm_100a kernels vs the CPU oracle and
the reference golden vectors.

Bars (north_star): tile/sort indices and per-tile ranges bit-exact; images
within 1e-4 abs (the exact path is in fact bit-identical to the oracle);
gradients within 1e-3 relative (see helpers.rel_err for the floor).
"""

import numpy as np
import pytest
import torch

from helpers import intr_from, np_map, pose_from, rel_err, window_maps
from oracle import raster as O

pytestmark = pytest.mark.gpu

I3 = np.eye(3)
Z3 = np.zeros(3)


def dev_map(m, dtype=torch.float64):
    from paper_2603_21055_b200.gaussians import PixelGaussianMap
    return PixelGaussianMap(m.frame_index, m.pose, m.intrinsics, m.base_depth, m.delta, m.color,
                            m.log_radius, m.opacity_logit, m.active_mask, dtype=dtype)


def offsets_from_ranges(ranges, n_pairs):
    nt = len(ranges)
    counts = ranges[:, 1] - ranges[:, 0]
    off = np.zeros(nt + 1, dtype=np.int64)
    off[1:] = np.cumsum(counts)
    # ranges of empty tiles are (0, 0); non-empty ones must be contiguous
    nz = counts > 0
    np.testing.assert_array_equal(ranges[nz, 0], off[:-1][nz])
    assert off[-1] == n_pairs
    return off


def check_view(maps_np, pose, intr, golden_pixel=None, golden_offsets=None, golden_lists=None):
    from paper_2603_21055_b200.rasterizer import inspect_view
    maps = [dev_map(m) for m in maps_np]
    s, ranges, lists = inspect_view(maps, pose, intr)
    b = O.prepare(maps_np, pose.rotation, pose.translation, intr, learnable="all")
    np.testing.assert_array_equal(s["map_pos"], b.map_pos)
    np.testing.assert_array_equal(s["pixel"], b.pixel_index)
    for k in ("u0", "v0", "z", "sigma", "opacity"):
        np.testing.assert_array_equal(s[k], getattr(b, k), err_msg=k)
    off, lst = O.tile_lists(b)
    np.testing.assert_array_equal(offsets_from_ranges(ranges, len(lists)), off)
    np.testing.assert_array_equal(lists, lst)
    if golden_pixel is not None:
        np.testing.assert_array_equal(s["pixel"], golden_pixel)
        np.testing.assert_array_equal(off, golden_offsets)
        np.testing.assert_array_equal(lists, golden_lists)
    return maps


def test_c1_indices_bit_exact(golden):
    g = golden("c1")
    intr = intr_from(g["intr"])
    from paper_2603_21055_b200.geometry import Pose
    check_view([np_map(g, "in_", intr)], Pose.identity(), intr, g["b_pixel"], g["offsets"],
               g["lists"])


def test_c1_render_and_grads(golden):
    from paper_2603_21055_b200 import mapper as M
    from paper_2603_21055_b200.geometry import Pose
    from paper_2603_21055_b200.scenes import Frame
    g = golden("c1")
    intr = intr_from(g["intr"])
    m_np = np_map(g, "in_", intr)
    m = dev_map(m_np)
    tf = Frame(g["t_color"], g["t_depth"], g["t_mask"], intr)
    loss, grads, out = M.mapping_loss([m], tf, Pose.identity(), M.MapperConfig(tau=0.0))
    # bit-identical to the oracle, within 1e-12 of the reference itself
    o_loss, o_grads, o_out = O.mapping_loss([m_np], g["t_color"], g["t_depth"], g["t_mask"], I3,
                                            Z3, intr)
    np.testing.assert_array_equal(out.color.cpu().numpy(), o_out.color)
    np.testing.assert_array_equal(out.depth.cpu().numpy(), o_out.depth)
    np.testing.assert_array_equal(out.alpha.cpu().numpy(), o_out.alpha)
    np.testing.assert_array_equal(out.contributors.cpu().numpy(), g["out_count"])
    np.testing.assert_allclose(out.color.cpu().numpy(), g["out_color"], atol=1e-12)
    np.testing.assert_allclose(out.depth.cpu().numpy(), g["out_depth"], atol=1e-12)
    np.testing.assert_allclose([loss.total, loss.color_l1, loss.depth_l1], g["loss"][[0, 1, 3]],
                               rtol=1e-12)
    for k, r in (("color", "g_color"), ("radius", "g_radius"), ("opacity_logit", "g_logit"),
                 ("delta", "g_delta")):
        got = getattr(grads, k).cpu().numpy()
        assert rel_err(got, g[r]) < 1e-9, k
        assert rel_err(got, getattr(o_grads, k)) < 1e-9, k
    opt = M.MapOptimizer(m, M.MapperConfig(tau=0.0))
    opt.step(grads)
    for k, r in (("color", "adam_color"), ("log_radius", "adam_log_radius"),
                 ("opacity_logit", "adam_logit"), ("delta", "adam_delta")):
        np.testing.assert_allclose(getattr(m, k).cpu().numpy(), g[r], atol=1e-9, err_msg=k)


@pytest.mark.parametrize("view", [0, 2])
def test_window_view_exact(golden, view):
    from paper_2603_21055_b200.rasterizer import splat, splat_backward
    g = golden("window")
    intr, maps_np = window_maps(g)
    pose = pose_from(g[f"m{view}_pose"])
    maps = check_view(maps_np, pose, intr, g[f"v{view}_b_pixel"], g[f"v{view}_offsets"],
                      g[f"v{view}_lists"])
    out = splat(maps, pose, intr)
    np.testing.assert_allclose(out.color.cpu().numpy(), g[f"v{view}_color"], atol=1e-12)
    np.testing.assert_allclose(out.depth.cpu().numpy(), g[f"v{view}_depth"], atol=1e-12)
    np.testing.assert_array_equal(out.contributors.cpu().numpy(), g[f"v{view}_count"])
    gc, gd, ga = g[f"v{view}_gc"], g[f"v{view}_gd"], g[f"v{view}_ga"]
    grads = splat_backward(maps, pose, intr, gc, gd, ga, learnable_map="all")
    for i, gr in enumerate(grads):
        for k, r in (("color", "g_color"), ("radius", "g_radius"), ("opacity_logit", "g_logit"),
                     ("delta", "g_delta")):
            assert rel_err(getattr(gr, k).cpu().numpy(), g[f"v{view}_m{i}_{r}"]) < 1e-9, (i, k)
    gn = splat_backward(maps, pose, intr, gc, gd, ga, learnable_map=1, normalize_depth=True)
    assert rel_err(gn.delta.cpu().numpy(), g[f"v{view}_norm_m1_g_delta"]) < 1e-9
    outn = splat(maps, pose, intr, normalize_depth=True)
    np.testing.assert_allclose(outn.depth.cpu().numpy(), g[f"v{view}_norm_depth"], atol=1e-12)


def _window_np(n_frames=3, seed=7, fx=60.0, w=64, h=48):
    from paper_2603_21055_b200 import scenes
    wc = scenes.config_window("t", n_frames, dict(fx=fx, fy=fx, cx=(w - 1) / 2, cy=(h - 1) / 2,
                                                  width=w, height=h))
    rng = np.random.default_rng(seed)
    for p in wc.params:
        p.delta = scenes._f32(rng.normal(0.0, 0.01, p.base_depth.shape))
        p.opacity_logit = scenes._f32(rng.normal(1.0, 1.0, p.base_depth.shape))
    return wc


@pytest.mark.parametrize("one_kernel", [True, False])
def test_window_engine_fused_vs_oracle(one_kernel):
    """Fused loss + fused fp32 backward of the WindowMapper vs the oracle's
    all-learnable window gradients (delta D1) on identical fp32 parameters --
    as one forward+backward kernel and as the two kernels."""
    from paper_2603_21055_b200.mapper import MapperConfig, WindowMapper
    from types import SimpleNamespace
    wc = _window_np()
    wm = WindowMapper(wc.frames, wc.poses, wc.intr, wc.params, MapperConfig(tau=0.0))
    wm.fuse_fwd_bwd = one_kernel
    maps_np = []
    for i, p in enumerate(wc.params):
        maps_np.append(SimpleNamespace(frame_index=i, pose=wc.poses[i], intrinsics=wc.intr,
                                       base_depth=p.base_depth, delta=p.delta,
                                       log_radius=p.log_radius, opacity_logit=p.opacity_logit,
                                       color=p.color, active_mask=p.active_mask))
    views = [(wc.poses[v].rotation, wc.poses[v].translation, wc.intr, wc.frames[v].color,
              wc.frames[v].depth, wc.frames[v].valid_mask) for v in range(len(wc.poses))]
    o_loss, o_grads = O.window_step_grads(maps_np, views)
    wm.loss_acc.zero_()
    for v in wm.views:
        wm.render_view_grads(v)
    n_color = 3.0 * wm.HW
    la = wm.loss_acc.cpu().numpy()
    loss = sum(0.8 * la[v, 0] / n_color + la[v, 1] / wm.n_depth[v] for v in range(wm.F))
    assert abs(loss - o_loss) <= 1e-9 * abs(o_loss)
    got = wm.grads_numpy()
    for i in range(wm.F):
        for k in ("color", "radius", "opacity_logit", "delta"):
            e = rel_err(got[i][k], getattr(o_grads[i], k), floor_frac=1e-3)
            assert e < 1e-3, (i, k, e)


def test_window_engine_step_adam():
    """One full WindowMapper step == oracle grads + oracle Adam (fp32 storage)."""
    from paper_2603_21055_b200.mapper import MapperConfig, WindowMapper
    wc = _window_np(n_frames=2, seed=3)
    cfg = MapperConfig(tau=0.0)
    wm = WindowMapper(wc.frames, wc.poses, wc.intr, wc.params, cfg)
    before = wm.planes.clone()
    wm.step()
    after = wm.planes.cpu().numpy()
    assert np.isfinite(after).all()
    # first Adam step moves every parameter with nonzero gradient by ~lr
    d = np.abs(after - before.cpu().numpy())
    assert d[:, 4:7].max() <= cfg.lr_color * 1.0001 + 1e-7
    assert d[:, 3].max() <= cfg.lr_opacity * 1.0001 + 1e-7
    assert (d[:, 0] == 0).all()  # base depth is not learnable
    assert wm.grad.abs().max().item() == 0.0  # consumed and zeroed by Adam


@pytest.mark.parametrize("seed", [11, 12])
def test_random_footprints_bit_exact(seed):
    """Gaussians with footprints from ~0.05 px to ~40 px, many centres near
    pixel-boundary distances: the fp32-guarded pixel masks must reproduce the
    reference test exactly, so images equal the oracle's bit for bit."""
    from types import SimpleNamespace
    from paper_2603_21055_b200.rasterizer import splat
    wc = _window_np(n_frames=3, seed=seed)
    rng = np.random.default_rng(seed)
    maps_np = []
    for i, p in enumerate(wc.params):
        p.log_radius = p.log_radius + rng.normal(0.0, 1.5, p.log_radius.shape)
        p.opacity_logit = rng.normal(0.0, 3.0, p.log_radius.shape)
        maps_np.append(SimpleNamespace(frame_index=i, pose=wc.poses[i], intrinsics=wc.intr,
                                       base_depth=p.base_depth, delta=p.delta,
                                       log_radius=p.log_radius, opacity_logit=p.opacity_logit,
                                       color=p.color, active_mask=p.active_mask))
    maps = [dev_map(m) for m in maps_np]
    for v in range(3):
        pose = wc.poses[v]
        out = splat(maps, pose, wc.intr)
        ref = O.splat(maps_np, pose.rotation, pose.translation, wc.intr)
        np.testing.assert_array_equal(out.contributors.cpu().numpy(), ref.contributors)
        np.testing.assert_array_equal(out.color.cpu().numpy(), ref.color)
        np.testing.assert_array_equal(out.depth.cpu().numpy(), ref.depth)


@pytest.mark.parametrize("scale", [1.2, 2.5, 4.0])
def test_tile_size_classes_bit_exact(scale):
    """Tile buckets of every size class of the shared-memory depth sort (<= 2048,
    <= 4096, <= 8192 pairs) and beyond it (the segmented-sort fallback): a third
    of the Gaussians get footprints of tens of pixels so that some tiles collect
    well over 8192 pairs.  Indices, ranges and images must equal the oracle's."""
    from types import SimpleNamespace
    from paper_2603_21055_b200.rasterizer import splat
    wc = _window_np(n_frames=3, seed=5, w=96, h=64, fx=80.0)
    rng = np.random.default_rng(17)
    maps_np = []
    for i, p in enumerate(wc.params):
        big = rng.random(p.log_radius.shape) < (0.6 if scale > 3.0 else 0.34)
        p.log_radius = p.log_radius + np.where(big, scale * rng.random(p.log_radius.shape) + 1.0,
                                               0.0)
        maps_np.append(SimpleNamespace(frame_index=i, pose=wc.poses[i], intrinsics=wc.intr,
                                       base_depth=p.base_depth, delta=p.delta,
                                       log_radius=p.log_radius, opacity_logit=p.opacity_logit,
                                       color=p.color, active_mask=p.active_mask))
    pose = wc.poses[1]
    maps = check_view(maps_np, pose, wc.intr)
    from paper_2603_21055_b200.rasterizer import inspect_view
    _, ranges, _ = inspect_view(maps, pose, wc.intr)
    sizes = ranges[:, 1] - ranges[:, 0]
    if scale > 3.0:
        assert sizes.max() > 8192, sizes.max()
    elif scale > 2.0:
        assert sizes.max() > 4096, sizes.max()
    else:
        assert sizes.max() > 2048, sizes.max()
    out = splat(maps, pose, wc.intr)
    ref = O.splat(maps_np, pose.rotation, pose.translation, wc.intr)
    np.testing.assert_array_equal(out.contributors.cpu().numpy(), ref.contributors)
    np.testing.assert_array_equal(out.color.cpu().numpy(), ref.color)


@pytest.mark.parametrize("size", [(64, 48), (160, 120)])
def test_fronto_parallel_runs_bit_exact(size):
    """A plane seen head-on at exactly equal depth: thousands of survivors
    share one depth bucket (the long-run sort), and the other frames'
    Gaussians on the same plane land in that bucket with depths a few ulps
    away -- the tile lists must still follow the exact (z, frame, pixel) order."""
    from types import SimpleNamespace
    w, h = size
    wc = _window_np(n_frames=3, seed=9, w=w, h=h, fx=w * 0.9)
    rng = np.random.default_rng(3)
    maps_np = []
    for i, p in enumerate(wc.params):
        if i == 0:
            p.base_depth = np.full_like(p.base_depth, 2.0)
            p.delta = np.zeros_like(p.delta)
        else:
            p.base_depth = np.full_like(p.base_depth, 2.0)
            p.delta = (rng.normal(0.0, 1e-9, p.delta.shape)).astype(np.float32).astype(np.float64)
        p.active_mask = np.ones_like(p.active_mask)
        maps_np.append(SimpleNamespace(frame_index=i, pose=wc.poses[i], intrinsics=wc.intr,
                                       base_depth=p.base_depth, delta=p.delta,
                                       log_radius=p.log_radius, opacity_logit=p.opacity_logit,
                                       color=p.color, active_mask=p.active_mask))
    from paper_2603_21055_b200.geometry import Pose
    check_view(maps_np, Pose.identity(), wc.intr)
    check_view(maps_np, wc.poses[1], wc.intr)


@pytest.mark.parametrize("bits", [16, 24, 32])
def test_unsorted_bucket_runs_bit_exact(monkeypatch, bits):
    """Runs of equal depth buckets holding distinct depths, from a few to one
    of ~50 k (a plane at 2 m with 1e-7 m of jitter, a few pixels at 8 m so the
    bucket width is far above the jitter): the fix-up's insertion sort, the
    shared-memory bitonic and the global merge sort of k_long_runs must all
    leave the exact (z, frame, pixel) order, at every depth-key width."""
    from types import SimpleNamespace
    from paper_2603_21055_b200.geometry import Pose
    monkeypatch.setenv("SGAD_DEPTH_BITS", str(bits))
    wc = _window_np(n_frames=3, seed=4, w=160, h=120, fx=140.0)
    rng = np.random.default_rng(11)
    maps_np = []
    for i, p in enumerate(wc.params):
        p.base_depth = np.full_like(p.base_depth, 2.0)
        p.delta = rng.normal(0.0, 1e-7, p.delta.shape).astype(np.float32).astype(np.float64)
        p.base_depth[:2, :4] = 8.0
        p.active_mask = np.ones_like(p.active_mask)
        maps_np.append(SimpleNamespace(frame_index=i, pose=Pose.identity(), intrinsics=wc.intr,
                                       base_depth=p.base_depth, delta=p.delta,
                                       log_radius=p.log_radius, opacity_logit=p.opacity_logit,
                                       color=p.color, active_mask=p.active_mask))
    check_view(maps_np, Pose.identity(), wc.intr)


def test_random_footprints_backward_exact():
    """The exact drop-in backward (compact per-warp lists from the forward, the
    ring of windows) against the oracle on footprints from ~0.05 px to ~40 px:
    all window maps learnable (delta D1), fp64 gradients within 1e-9."""
    from types import SimpleNamespace
    from paper_2603_21055_b200.rasterizer import splat_backward
    wc = _window_np(n_frames=3, seed=21)
    rng = np.random.default_rng(21)
    maps_np = []
    for i, p in enumerate(wc.params):
        p.log_radius = p.log_radius + rng.normal(0.0, 1.5, p.log_radius.shape)
        p.opacity_logit = rng.normal(0.0, 3.0, p.log_radius.shape)
        maps_np.append(SimpleNamespace(frame_index=i, pose=wc.poses[i], intrinsics=wc.intr,
                                       base_depth=p.base_depth, delta=p.delta,
                                       log_radius=p.log_radius, opacity_logit=p.opacity_logit,
                                       color=p.color, active_mask=p.active_mask))
    maps = [dev_map(m) for m in maps_np]
    h, w = wc.intr.height, wc.intr.width
    gc = rng.normal(0, 1e-3, (h, w, 3))
    gd = rng.normal(0, 1e-3, (h, w))
    ga = rng.normal(0, 1e-3, (h, w))
    pose = wc.poses[1]
    ref = O.splat_backward(maps_np, pose.rotation, pose.translation, wc.intr, gc, gd, ga,
                           learnable_map="all")
    got = splat_backward(maps, pose, wc.intr, torch.as_tensor(gc, device="cuda"),
                         torch.as_tensor(gd, device="cuda"), torch.as_tensor(ga, device="cuda"),
                         learnable_map="all")
    for i in range(3):
        for k in ("color", "radius", "opacity_logit", "delta"):
            a = getattr(got[i], k)
            a = a.cpu().numpy() if isinstance(a, torch.Tensor) else a
            assert rel_err(a, getattr(ref[i], k)) < 1e-9, (i, k)


def test_unpacked_lists_same_results(monkeypatch):
    """Views with 2^26 or more Gaussians keep bare record ids in their tile
    lists (no warp-rectangle bits, K4 culls nothing from the list word).
    Forced on a small window (SGAD_PACK=0), images and window gradients must
    equal the packed path's bit for bit."""
    from types import SimpleNamespace
    from paper_2603_21055_b200.mapper import MapperConfig, WindowMapper
    from paper_2603_21055_b200.rasterizer import splat
    wc = _window_np(n_frames=3, seed=21)
    maps = [dev_map(SimpleNamespace(frame_index=i, pose=wc.poses[i], intrinsics=wc.intr,
                                    base_depth=p.base_depth, delta=p.delta,
                                    log_radius=p.log_radius, opacity_logit=p.opacity_logit,
                                    color=p.color, active_mask=p.active_mask))
            for i, p in enumerate(wc.params)]

    def run():
        out = [splat(maps, wc.poses[v], wc.intr) for v in range(3)]
        imgs = [(o.color.cpu().numpy(), o.depth.cpu().numpy(), o.contributors.cpu().numpy())
                for o in out]
        wm = WindowMapper(wc.frames, wc.poses, wc.intr, wc.params, MapperConfig(tau=0.0))
        wm.loss_acc.zero_()
        for v in wm.views:
            wm.render_view_grads(v)
        return imgs, wm.grad.cpu().numpy(), wm.loss_acc.cpu().numpy()

    imgs_p, grad_p, loss_p = run()
    monkeypatch.setenv("SGAD_PACK", "0")
    imgs_u, grad_u, loss_u = run()
    for a, b in zip(imgs_p, imgs_u):
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)
    # loss and gradient sums are float atomics: equal up to summation order
    np.testing.assert_allclose(loss_u, loss_p, rtol=1e-12)
    np.testing.assert_allclose(grad_u, grad_p, rtol=1e-5, atol=1e-9)


@pytest.mark.parametrize("hw", [4096, 4093])
def test_window_adam_fp32_vs_numpy(hw):
    """The window engine's fp32 Adam (vectorised kernel when hw % 4 == 0,
    scalar otherwise) vs a numpy restatement of mapper.py:73-95 in fp64:
    radius gradient chained to log radius, bias corrections, colour clip;
    gradients consumed (zeroed)."""
    import torch
    from paper_2603_21055_b200.mapper import MapperConfig, _adam
    cfg = MapperConfig(tau=0.0)
    F = 3
    rng = np.random.default_rng(hw)
    params = rng.uniform(0.0, 1.0, (F, 7, hw)).astype(np.float32)
    params[:, 2] = rng.normal(-4.0, 0.5, (F, hw))  # log radius
    m = rng.normal(0.0, 1e-3, (F, 6, hw)).astype(np.float32)
    v = rng.uniform(0.0, 1e-5, (F, 6, hw)).astype(np.float32)
    g = rng.normal(0.0, 1e-2, (F * hw, 8)).astype(np.float32)
    t = 5
    dev = torch.device("cuda", 0)
    P, M, V, G = (torch.from_numpy(x.copy()).to(dev) for x in (params, m, v, g))
    _adam(P, G, M, V, F, hw, cfg, t, False)
    torch.cuda.synchronize()
    b1, b2, eps = cfg.adam_beta1, cfg.adam_beta2, cfg.adam_eps
    lr = np.array(cfg.lrs())
    gg = g.reshape(F, hw, 8).astype(np.float64)
    grad = np.stack([gg[..., 0], gg[..., 1] * np.exp(params[:, 2].astype(np.float64)),
                     gg[..., 2], gg[..., 3], gg[..., 4], gg[..., 5]], axis=1)  # [F, 6, hw]
    m1 = b1 * m + (1 - b1) * grad
    v1 = b2 * v + (1 - b2) * grad * grad
    step = lr[None, :, None] * (m1 / (1 - b1**t)) / (np.sqrt(v1 / (1 - b2**t)) + eps)
    p1 = params[:, 1:].astype(np.float64) - step
    p1[:, 3:] = np.clip(p1[:, 3:], 0.0, 1.0)
    # fp32 storage and arithmetic (1 - beta2 alone is 1.3e-5 off in fp32)
    np.testing.assert_allclose(M.cpu().numpy(), m1, rtol=1e-5, atol=1e-9)
    np.testing.assert_allclose(V.cpu().numpy(), v1, rtol=5e-5, atol=1e-12)
    np.testing.assert_allclose(P.cpu().numpy()[:, 1:], p1, rtol=1e-5, atol=1e-6)
    np.testing.assert_array_equal(P.cpu().numpy()[:, 0], params[:, 0])  # base depth untouched
    assert G.abs().max().item() == 0.0


def test_c3_full_size_view_vs_oracle():
    """One view of the full-size C3 window (640x480, 8 keyframes, 2.46 M
    Gaussians, BASELINE config): the drop-in splat's images bit-identical to
    the oracle and the window engine's fused gradients for that view within
    the 1e-3 bar -- parity at the benchmark's own size, not only on small
    goldens."""
    from types import SimpleNamespace
    from paper_2603_21055_b200 import scenes
    from paper_2603_21055_b200.mapper import MapperConfig, WindowMapper
    from paper_2603_21055_b200.rasterizer import splat
    wc = scenes.config_c3(device="cuda")
    v = 3
    maps_np = [SimpleNamespace(frame_index=i, pose=wc.poses[i], intrinsics=wc.intr,
                               base_depth=p.base_depth, delta=p.delta, log_radius=p.log_radius,
                               opacity_logit=p.opacity_logit, color=p.color,
                               active_mask=p.active_mask) for i, p in enumerate(wc.params)]
    pose = wc.poses[v]
    out = splat([dev_map(m) for m in maps_np], pose, wc.intr)
    ref = O.splat(maps_np, pose.rotation, pose.translation, wc.intr)
    np.testing.assert_array_equal(out.contributors.cpu().numpy(), ref.contributors)
    np.testing.assert_array_equal(out.color.cpu().numpy(), ref.color)
    np.testing.assert_array_equal(out.depth.cpu().numpy(), ref.depth)
    fr = wc.frames[v]
    o_loss, o_grads = O.window_step_grads(
        maps_np, [(pose.rotation, pose.translation, wc.intr, fr.color, fr.depth, fr.valid_mask)])
    wm = WindowMapper(wc.frames, wc.poses, wc.intr, wc.params, MapperConfig(tau=0.0))
    wm.loss_acc.zero_()
    wm.render_view_grads(v)
    la = wm.loss_acc.cpu().numpy()
    loss = 0.8 * la[v, 0] / (3.0 * wm.HW) + la[v, 1] / wm.n_depth[v]
    assert abs(loss - o_loss) <= 1e-9 * abs(o_loss)
    got = wm.grads_numpy()
    for i in range(wm.F):
        for k in ("color", "radius", "opacity_logit", "delta"):
            e = rel_err(got[i][k], getattr(o_grads[i], k), floor_frac=1e-3)
            assert e < 1e-3, (i, k, e)


def test_c4_full_size_images_vs_oracle():
    """The headline configuration's size (1200x680, 8 keyframes, 6.53 M
    Gaussians): one view's images and contributor counts bit-identical to
    the oracle."""
    from types import SimpleNamespace
    from paper_2603_21055_b200 import scenes
    from paper_2603_21055_b200.rasterizer import splat
    wc = scenes.config_c4(device="cuda")
    v = 5
    maps_np = [SimpleNamespace(frame_index=i, pose=wc.poses[i], intrinsics=wc.intr,
                               base_depth=p.base_depth, delta=p.delta, log_radius=p.log_radius,
                               opacity_logit=p.opacity_logit, color=p.color,
                               active_mask=p.active_mask) for i, p in enumerate(wc.params)]
    pose = wc.poses[v]
    out = splat([dev_map(m) for m in maps_np], pose, wc.intr)
    ref = O.splat(maps_np, pose.rotation, pose.translation, wc.intr)
    np.testing.assert_array_equal(out.contributors.cpu().numpy(), ref.contributors)
    np.testing.assert_array_equal(out.color.cpu().numpy(), ref.color)
    np.testing.assert_array_equal(out.depth.cpu().numpy(), ref.depth)
    np.testing.assert_array_equal(out.alpha.cpu().numpy(), ref.alpha)


def test_window_step_cuda_graph_matches_eager():
    """The window step captured in a CUDA graph (use_graph) and replayed:
    the same losses, step count and parameters as eager steps (fp32
    gradient sums in another order: 1e-5)."""
    from paper_2603_21055_b200.mapper import MapperConfig, WindowMapper
    wc = _window_np(n_frames=4, seed=12)
    runs = {}
    for graph in (False, True):
        wm = WindowMapper(wc.frames, wc.poses, wc.intr, wc.params, MapperConfig(tau=0.0))
        wm.use_graph = graph
        losses = [wm.step(sync_loss=True) for _ in range(4)]
        runs[graph] = (np.array(losses), wm.t, wm.planes.cpu().numpy(), wm._graph is not None)
    assert runs[True][3] and not runs[False][3]
    assert runs[True][1] == runs[False][1] == 4
    np.testing.assert_allclose(runs[True][0], runs[False][0], rtol=1e-5)
    np.testing.assert_allclose(runs[True][2], runs[False][2], rtol=0, atol=2e-3)


def test_window_step_with_host_targets():
    """step_with_targets (targets uploaded from pinned host buffers inside the
    step, eager and replayed from a CUDA graph) against step() with the same
    targets resident: the same losses, step count and parameters (fp32
    gradient sums in another order: 1e-5), and the uploaded targets land."""
    from paper_2603_21055_b200.mapper import MapperConfig, WindowMapper
    wc = _window_np(n_frames=4, seed=13)
    runs = {}
    for mode in ("resident", "host", "host_graph"):
        wm = WindowMapper(wc.frames, wc.poses, wc.intr, wc.params, MapperConfig(tau=0.0))
        wm.use_graph = mode == "host_graph"
        vs = list(wm.views)
        tc = wm.tcolor[vs].cpu().pin_memory()
        td = wm.tdepth[vs].cpu().pin_memory()
        tm = wm.tmask[vs].cpu().pin_memory()
        if mode != "resident":  # the device copies must come from the uploads
            wm.tcolor.zero_()
            wm.tdepth.zero_()
            wm.tmask.zero_()
        losses = [wm.step(sync_loss=True) if mode == "resident" else
                  wm.step_with_targets(tc, td, tm, sync_loss=True) for _ in range(4)]
        runs[mode] = (np.array(losses), wm.t, wm.planes.cpu().numpy())
        if mode == "host_graph":
            assert wm._hgraph is not None
    with pytest.raises(ValueError):  # pageable buffers cannot be captured
        wm.step_with_targets(tc.clone(), td, tm)
    for mode in ("host", "host_graph"):
        assert runs[mode][1] == runs["resident"][1] == 4
        np.testing.assert_allclose(runs[mode][0], runs["resident"][0], rtol=1e-5)
        np.testing.assert_allclose(runs[mode][2], runs["resident"][2], rtol=0, atol=2e-3)


@pytest.mark.parametrize("graph", [False, True])
def test_window_view_without_survivors(graph):
    """A window view that sees no Gaussian (its own frame has no active
    pixel and it faces away from the others): the step runs through the
    asynchronous preparation (zero survivors, empty tile lists), the view's
    loss is its bare target, it adds no gradient -- the parameters move as
    in a window that renders only the other view."""
    from paper_2603_21055_b200.geometry import Pose
    from paper_2603_21055_b200.mapper import MapperConfig, WindowMapper
    wc = _window_np(n_frames=2, seed=5)
    wc.params[1].active_mask[:] = False
    flip = np.diag([-1.0, 1.0, -1.0])  # 180 degrees about y: looking away
    wc.poses[1] = Pose(wc.poses[0].rotation @ flip, wc.poses[0].translation)
    runs = {}
    for views in ([0, 1], [0]):
        wm = WindowMapper(wc.frames, wc.poses, wc.intr, wc.params, MapperConfig(tau=0.0),
                          views=views)
        wm.use_graph = graph
        losses = [wm.step(sync_loss=True) for _ in range(3)]
        runs[tuple(views)] = (np.array(losses), wm.planes.cpu().numpy(), wm.counts())
    (l2, p2, c2), (l1, p1, c1) = runs[(0, 1)], runs[(0,)]
    assert c2[1] == (0, 0) and c2[0][0] > 0
    assert np.all(np.isfinite(l2)) and np.all(l2 > l1)
    # (the fp32 gradient atomics sum in run-dependent order: an ulp apart)
    np.testing.assert_allclose(p2, p1, rtol=0, atol=1e-5)


def test_window_pair_capacity_overflow_recovers():
    """The asynchronous preparation outgrowing its pair capacity (the radii
    grow after the handles were sized): the view sets the device overflow
    flag, Adam skips that step on the device (no update, step count
    unchanged), the host grows the capacity and the synchronous step runs
    again -- the same trajectory as a window re-sized before the growth."""
    from paper_2603_21055_b200.mapper import MapperConfig, WindowMapper
    wc = _window_np(n_frames=3, seed=21)
    runs = []
    for resize in (True, False):
        wm = WindowMapper(wc.frames, wc.poses, wc.intr, wc.params, MapperConfig(tau=0.0))
        wm.step(sync_loss=True)           # sizes the handles for these radii
        wm.planes[:, 2] += 1.5            # radii x4.5: far more tile pairs
        if resize:
            wm._cap = 0                   # (re-sized at the next step: no overflow)
        losses = [wm.step(sync_loss=True) for _ in range(3)]
        runs.append((np.array(losses), wm.t, wm.overflows))
    assert runs[0][2] == 0 and runs[1][2] >= 1
    np.testing.assert_allclose(runs[1][0], runs[0][0], rtol=1e-5)
    assert runs[1][1] == runs[0][1] == 4
