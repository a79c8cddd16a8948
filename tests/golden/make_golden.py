"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py [c1 window eig track ssim render_init voxels frame_driver]

The reference package is copied to a temporary directory first (so nothing is
written under /root/reference: Numba's cache and __pycache__ land in the
copy) and imported from there.  The inputs are produced by this repo's seeded
scene generator and handed to the reference as plain arrays, so the goldens
pin the reference's arithmetic only.  The resulting .npz files are committed;
tests and the oracle read them on machines without /root/reference.
"""

from __future__ import annotations

import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src/raysplat"


def import_reference():
    tmp = tempfile.mkdtemp(prefix="raysplat_ref_")
    shutil.copytree(REF_SRC, os.path.join(tmp, "raysplat"))
    os.environ["NUMBA_CACHE_DIR"] = os.path.join(tmp, "numba_cache")
    sys.dont_write_bytecode = True
    sys.path.insert(0, tmp)
    import raysplat.gaussians as G  # noqa: E402
    import raysplat.geometry as GEO
    import raysplat.mapper as M
    import raysplat.rasterizer as R
    import raysplat.tracker as T
    from raysplat.datasets import RgbdFrame
    return tmp, G, GEO, M, R, T, RgbdFrame


def golden_ssim(M, G, GEO, R, RgbdFrame):
    """raysplat/ssim.py on seeded image pairs (3-channel, 1-channel, a
    constant pair, tiny and odd sizes) and the full tau = 0.2 mapping_loss of
    configuration C1 (mapper.py:106-157 with the SSIM term)."""
    import raysplat.ssim as S
    from paper_2603_21055_b200 import scenes
    rng = np.random.default_rng(2024)
    d = {}
    cases = {
        "rgb": (rng.random((45, 61, 3)), None),
        "gray": (rng.random((23, 17)), None),
        "const": (np.full((12, 14, 3), 0.3), np.full((12, 14, 3), 0.7)),
        "tiny": (rng.random((4, 6, 3)), None),
    }
    for name, (a, b) in cases.items():
        if b is None:
            b = np.clip(a + rng.normal(0.0, 0.15, a.shape), 0.0, 1.0)
        v, g = S.ssim(a, b, with_grad=True)
        d[f"{name}_a"], d[f"{name}_b"] = a, b
        d[f"{name}_value"], d[f"{name}_grad"] = np.array(v), g
    intr, frame, learn, target = scenes.config_c1()
    ri = ref_intr(GEO, intr)
    ident = GEO.Pose.identity()
    m_learn = ref_map(G, GEO, learn, ri, ident, 0)
    m_tgt = ref_map(G, GEO, target, ri, ident, 0)
    t_out = R.splat([m_tgt], ident, ri)
    t_color = np.clip(t_out.color, 0.0, 1.0).astype(np.float32)
    t_depth = t_out.depth.astype(np.float32)
    tf = RgbdFrame(color=t_color, depth=t_depth, valid_mask=frame.valid_mask.copy(),
                   intrinsics=ri, timestamp=0.0, index=0)
    cfg = M.MapperConfig(tau=0.2)
    loss, grads, out = M.mapping_loss([m_learn], tf, ident, cfg)
    d["c1_loss"] = np.array([loss.total, loss.color_l1, loss.ssim_term, loss.depth_l1])
    d["c1_g_color"], d["c1_g_radius"] = grads.color, grads.radius
    d["c1_g_logit"], d["c1_g_delta"] = grads.opacity_logit, grads.delta
    d["c1_t_color"], d["c1_t_depth"], d["c1_t_mask"] = t_color, t_depth, frame.valid_mask
    return d


def ref_map(G, GEO, params, intr_ref, pose, frame_index):
    return G.PixelGaussianMap(
        frame_index=frame_index, pose=GEO.Pose(pose.rotation, pose.translation),
        intrinsics=intr_ref, base_depth=params.base_depth.copy(), delta=params.delta.copy(),
        color=params.color.copy(), log_radius=params.log_radius.copy(),
        opacity_logit=params.opacity_logit.copy(), active_mask=params.active_mask.copy())


def ref_intr(GEO, intr):
    return GEO.Intrinsics(fx=intr.fx, fy=intr.fy, cx=intr.cx, cy=intr.cy, width=intr.width,
                          height=intr.height)


def params_dict(prefix, p):
    return {f"{prefix}base_depth": p.base_depth, f"{prefix}delta": p.delta,
            f"{prefix}log_radius": p.log_radius, f"{prefix}opacity_logit": p.opacity_logit,
            f"{prefix}color": p.color, f"{prefix}active_mask": p.active_mask}


def golden_c1(G, GEO, M, R, RgbdFrame):
    from paper_2603_21055_b200 import scenes
    intr, frame, learn, target = scenes.config_c1()
    ri = ref_intr(GEO, intr)
    ident = GEO.Pose.identity()
    m_learn = ref_map(G, GEO, learn, ri, ident, 0)
    m_tgt = ref_map(G, GEO, target, ri, ident, 0)
    t_out = R.splat([m_tgt], ident, ri)
    t_color = np.clip(t_out.color, 0.0, 1.0).astype(np.float32)
    t_depth = t_out.depth.astype(np.float32)
    t_mask = frame.valid_mask.copy()
    tf = RgbdFrame(color=t_color, depth=t_depth, valid_mask=t_mask, intrinsics=ri, timestamp=0.0,
                   index=0)
    cfg = M.MapperConfig(tau=0.0)
    loss, grads, out = M.mapping_loss([m_learn], tf, ident, cfg)
    batch = R._prepare([m_learn], ident, ri, learnable_map=0)
    offsets, lists = R._build_tile_lists(batch.u0, batch.v0, batch.sigma, intr.height,
                                         intr.width, R._TILE)
    opt = M.MapOptimizer(m_learn, cfg)
    opt.step(grads)
    d = params_dict("in_", learn)
    d.update(t_color=t_color, t_depth=t_depth, t_mask=t_mask,
             intr=np.array([intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height]),
             loss=np.array([loss.total, loss.color_l1, loss.ssim_term, loss.depth_l1]),
             out_color=out.color, out_depth=out.depth, out_alpha=out.alpha,
             out_count=out.contributors, g_color=grads.color, g_radius=grads.radius,
             g_logit=grads.opacity_logit, g_delta=grads.delta,
             b_u0=batch.u0, b_v0=batch.v0, b_z=batch.z, b_sigma=batch.sigma,
             b_opacity=batch.opacity, b_pixel=batch.pixel_index, offsets=offsets,
             lists=lists.astype(np.int32),
             adam_color=m_learn.color, adam_log_radius=m_learn.log_radius,
             adam_logit=m_learn.opacity_logit, adam_delta=m_learn.delta)
    return d


def golden_window(G, GEO, R):
    """Delta D1 window: 3 frames of 64x48, all learnable, 2 target views."""
    from paper_2603_21055_b200 import scenes
    intr_kw = dict(fx=60.0, fy=60.0, cx=31.5, cy=23.5, width=64, height=48)
    wc = scenes.config_window("golden", 3, intr_kw)
    rng = np.random.default_rng(7)
    params = []
    for p in wc.params:  # perturb so every attribute carries gradient
        h, w = p.base_depth.shape
        p.delta = scenes._f32(rng.normal(0.0, 0.01, (h, w)))
        p.opacity_logit = scenes._f32(rng.normal(1.0, 1.0, (h, w)))
        p.log_radius = scenes._f32(p.log_radius + rng.normal(0.0, 0.3, (h, w)))
        params.append(p)
    ri = ref_intr(GEO, wc.intr)
    maps = [ref_map(G, GEO, p, ri, wc.poses[i], i) for i, p in enumerate(params)]
    d = {}
    for i, p in enumerate(params):
        d.update(params_dict(f"m{i}_", p))
        d[f"m{i}_pose"] = np.concatenate([wc.poses[i].rotation.reshape(9),
                                          wc.poses[i].translation])
    d["intr"] = np.array([ri.fx, ri.fy, ri.cx, ri.cy, ri.width, ri.height])
    views = [0, 2]
    grng = np.random.default_rng(8)
    for v in views:
        pose = GEO.Pose(wc.poses[v].rotation, wc.poses[v].translation)
        batch = R._prepare(maps, pose, ri, learnable_map=0)
        offsets, lists = R._build_tile_lists(batch.u0, batch.v0, batch.sigma, ri.height, ri.width,
                                             R._TILE)
        out = R.splat(maps, pose, ri)
        gc = grng.normal(size=(ri.height, ri.width, 3))
        gd = grng.normal(size=(ri.height, ri.width))
        ga = grng.normal(size=(ri.height, ri.width))
        frame_of = np.concatenate([np.full(int(m.active_mask.sum()), m.frame_index) for m in maps])
        del frame_of
        d[f"v{v}_offsets"] = offsets
        d[f"v{v}_lists"] = lists.astype(np.int32)
        d[f"v{v}_b_pixel"] = batch.pixel_index
        d[f"v{v}_b_u0"], d[f"v{v}_b_v0"] = batch.u0, batch.v0
        d[f"v{v}_b_z"], d[f"v{v}_b_sigma"] = batch.z, batch.sigma
        d[f"v{v}_color"], d[f"v{v}_depth"] = out.color, out.depth
        d[f"v{v}_alpha"], d[f"v{v}_count"] = out.alpha, out.contributors
        d[f"v{v}_gc"], d[f"v{v}_gd"], d[f"v{v}_ga"] = gc, gd, ga
        for i in range(len(maps)):
            g = R.splat_backward(maps, pose, ri, gc, gd, ga, learnable_map=i)
            d[f"v{v}_m{i}_g_color"] = g.color
            d[f"v{v}_m{i}_g_radius"] = g.radius
            d[f"v{v}_m{i}_g_logit"] = g.opacity_logit
            d[f"v{v}_m{i}_g_delta"] = g.delta
        gn = R.splat_backward(maps, pose, ri, gc, gd, ga, learnable_map=1, normalize_depth=True)
        d[f"v{v}_norm_m1_g_delta"] = gn.delta
        d[f"v{v}_norm_m1_g_radius"] = gn.radius
        outn = R.splat(maps, pose, ri, normalize_depth=True)
        d[f"v{v}_norm_depth"] = outn.depth
    d["views"] = np.array(views)
    return d


def golden_eig(GEO):
    rng = np.random.default_rng(31)
    mats = []
    for _ in range(300):
        a = rng.normal(size=(3, 3))
        mats.append(a @ a.T + 1e-6 * np.eye(3))
    mats.append(np.diag([4.0, 1.0, 0.25]))
    mats.append(np.eye(3))
    mats.append(np.diag([2.0, 1.0, 0.0]))
    mats.append(np.diag([1.0, 1.0 + 1e-13, 2.0]))
    mats.append(np.diag([1.0, 0.5, -1e-12]))
    pts = rng.normal(size=(200, 24, 3)) * np.array([1.0, 0.3, 1e-4])
    for k in range(200):
        dd = pts[k] - pts[k].mean(0)
        mats.append(dd.T @ dd / 24.0)
    mats = np.array(mats)
    rot, vals = GEO.sym_eigh3_batch(mats)
    return dict(mats=mats, rot=rot, vals=vals)


def window_fit_ref(T, GEO, depth, mask, intr, win=5, k_min=4, scale_mode="ellipse"):
    """Delta D2 restated ONLY in the neighbour selection; the covariance line,
    eigensolver, floor, normalisation and orientation are the reference's own
    (tracker.py:158-169, geometry.py:275)."""
    h, w = depth.shape
    valid = np.asarray(mask, dtype=bool)  # tracker.py:201 uses valid_mask only
    vs, us = np.nonzero(valid)
    z_all = depth[vs, us].astype(np.float64)
    pts = np.zeros((h, w, 3))
    pts[vs, us] = np.stack([(us - intr.cx) / intr.fx * z_all, (vs - intr.cy) / intr.fy * z_all,
                            z_all], axis=1)
    r = win // 2
    centers, covs, idx = [], [], []
    for v, u in zip(vs, us):
        nb = []
        for dv in range(-r, r + 1):
            for du in range(-r, r + 1):
                if dv == 0 and du == 0:
                    continue
                y, x = v + dv, u + du
                if 0 <= y < h and 0 <= x < w and valid[y, x]:
                    nb.append(pts[y, x])
        if len(nb) < k_min:
            continue
        nbr = np.array(nb)[None]
        diff = nbr - nbr.mean(axis=1, keepdims=True)
        cov = np.einsum("nki,nkj->nij", diff, diff) / nbr.shape[1]
        covs.append(cov[0])
        centers.append(pts[v, u])
        idx.append(v * w + u)
    centers = np.array(centers)
    cov = np.array(covs)
    rot, vals = GEO.sym_eigh3_batch(cov)
    vals = np.maximum(vals, T.EIGVAL_FLOOR_REL * vals[:, :1])
    scales = T._normalize_scales(np.sqrt(vals), scale_mode)
    normals = rot[:, :, 2].copy()
    flip = np.einsum("ni,ni->n", normals, -centers) < 0.0
    normals[flip] *= -1.0
    rot[flip, :, 2] *= -1.0
    rot[flip, :, 1] *= -1.0
    return np.array(idx), centers, rot, scales, normals


def golden_track(T, GEO):
    from paper_2603_21055_b200 import scenes
    intr_kw = dict(fx=60.0, fy=60.0, cx=39.5, cy=29.5, width=80, height=60)
    intr = scenes.Intrinsics(**intr_kw)
    prims = scenes.plane_spheres_scene(0)
    rng = np.random.default_rng(3)
    axis = rng.normal(size=3)
    axis /= np.linalg.norm(axis)
    angle = rng.uniform(0.0, np.deg2rad(2.0))
    shift = rng.normal(size=3)
    shift = shift / np.linalg.norm(shift) * rng.uniform(0.0, 0.05)
    truth = scenes.Pose(scenes.se3_exp(np.concatenate([axis * angle, np.zeros(3)])).rotation, shift)
    ref = scenes.render_frame(prims, scenes.Pose.identity(), intr, 0, depth_noise_rel=0.01)
    qry = scenes.render_frame(prims, truth, intr, 1, depth_noise_rel=0.01)
    d = dict(ref_depth=ref.depth, ref_mask=ref.valid_mask, qry_depth=qry.depth,
             qry_mask=qry.valid_mask, intr=np.array([intr.fx, intr.fy, intr.cx, intr.cy,
                                                     intr.width, intr.height]),
             truth=np.concatenate([truth.rotation.reshape(9), truth.translation]))
    fits = {}
    for name, fr in (("ref", ref), ("qry", qry)):
        idx, c, rot, s, n = window_fit_ref(T, GEO, fr.depth, fr.valid_mask, intr)
        fits[name] = (c, rot, s, n)
        d.update({f"{name}_idx": idx, f"{name}_centers": c, f"{name}_rot": rot,
                  f"{name}_scales": s, f"{name}_normals": n})
    c, rot, s, n = fits["ref"]
    g = T.GlobalGeomSet(voxel_size=1e-4)
    added = g.insert(c, rot, s, n)
    assert added == len(c)
    c, rot, s, n = fits["qry"]
    local = T.LocalGeomSet(centers=c, rotations=rot, scales=s, normals=n)
    cfg = T.TrackerConfig(max_gicp_iters=20, convergence_eps=0.0)
    pose, diag = T.gicp_align(local, g, GEO.Pose.identity(), cfg)
    d.update(gicp_pose=np.concatenate([pose.rotation.reshape(9), pose.translation]),
             gicp_iters=np.array(diag.iterations), gicp_inliers=np.array(diag.inlier_count),
             gicp_cost_pairs=np.array(diag.cost_pairs), gicp_final_cost=np.array(diag.final_cost),
             gicp_accepted_first=diag.accepted_first)
    # the first iteration's normal equations, restated from tracker.py:286-321
    pts = local.centers.copy()
    dist, j = g.query_nearest(pts)
    b = g.centers[j]
    dd = b - pts
    metric = np.abs(np.einsum("ni,ni->n", g.normals[j], dd))
    acc = metric < cfg.correspondence_dist_max
    c_comb = g.covariances(j[acc]) + local.covariances()[acc]
    wts = np.linalg.inv(c_comb)
    p_acc = pts[acc]
    jac = np.concatenate([T._skew(p_acc), -np.broadcast_to(np.eye(3), (int(acc.sum()), 3, 3))], 2)
    d["first_H"] = np.einsum("nij,nik,nkl->jl", jac, wts, jac)
    d["first_g"] = np.einsum("nij,nik,nk->j", jac, wts, dd[acc])
    d["first_nn"] = j
    d["first_cost"] = np.array(float(np.einsum("ni,nij,nj->", dd[acc], wts, dd[acc])))
    return d


def golden_render_init(G, GEO, T, RgbdFrame):
    """tracker.py:354-426 (init_pose_render) on the C1 scene: the map of frame
    A against frame B under a seeded offset, from the identity, plus a
    low-coverage case (the map shifted out of view) that must return the
    initial pose with ok = False."""
    from paper_2603_21055_b200 import scenes
    intr, fa, fb, params, truth = scenes.config_render_init()
    ri = ref_intr(GEO, intr)
    ident = GEO.Pose.identity()
    m = ref_map(G, GEO, params, ri, ident, 0)
    tf = RgbdFrame(color=fb.color, depth=fb.depth, valid_mask=fb.valid_mask, intrinsics=ri,
                   timestamp=0.0, index=1)
    d = {"truth_R": truth.rotation, "truth_t": truth.translation}
    for iters in (1, 10):
        pose, ok = T.init_pose_render(tf, m, ident, iters=iters)
        d[f"it{iters}_R"], d[f"it{iters}_t"], d[f"it{iters}_ok"] = (pose.rotation,
                                                                   pose.translation, np.array(ok))
    far = GEO.Pose(np.eye(3), np.array([5.0, 0.0, 0.0]))
    pose, ok = T.init_pose_render(tf, m, far, iters=3)
    d["far_R"], d["far_t"], d["far_ok"] = pose.rotation, pose.translation, np.array(ok)
    return d


def golden_voxels(T):
    """GlobalGeomSet.insert (tracker.py:105-122) on seeded batches with many
    cell collisions (within and across batches, negative coordinates)."""
    rng = np.random.default_rng(31)
    g = T.GlobalGeomSet(voxel_size=0.05)
    d = {}
    for b in range(3):
        n = 4000
        c = rng.uniform(-1.0, 1.0, (n, 3)) * np.array([1.0, 0.5, 0.25])
        c[n // 2:] = c[: n - n // 2] + rng.normal(0, 0.01, (n - n // 2, 3))  # near-duplicates
        rot = np.repeat(np.eye(3)[None], n, axis=0)
        sc = rng.uniform(0.01, 0.1, (n, 3))
        nr = np.tile([0.0, 0.0, -1.0], (n, 1))
        added = g.insert(c, rot, sc, nr)
        d[f"b{b}_centers"], d[f"b{b}_scales"], d[f"b{b}_added"] = c, sc, np.array(added)
        d[f"b{b}_members"] = g.centers.copy()
    return d


def golden_frame_driver(G, GEO, M, RgbdFrame):
    """The per-frame mapping driver and its formats, from the reference:
    target_schedule (mapper.py:175-194), inpaint_depth (datasets.py:368-398),
    assemble_base_depth (:197-214), map_frame (:217-247, 4 iterations, tau
    0.2) and the .bin map file bytes (gaussians.py:118-136)."""
    import io
    import tempfile as _tf
    from raysplat.datasets import inpaint_depth
    from paper_2603_21055_b200 import scenes
    d = {}
    cases = [(10, 0, 0.4, 0), (25, 1, 0.4, 0), (40, 3, 0.4, 2), (17, 2, 0.7, 5), (9, 4, 0.0, 1)]
    for i, (it, n, frac, seed) in enumerate(cases):
        d[f"sched{i}"] = np.array(M.target_schedule(it, n, frac, seed))
        d[f"sched{i}_args"] = np.array([it, n, frac, seed])
    intr, fa, fb, params, truth = scenes.config_render_init()
    rng = np.random.default_rng(12)
    holes = rng.random(fb.depth.shape) < 0.05
    holes[40:70, 90:130] = True            # a block the neighbour covers
    holes[:, :6] = True                    # a border strip
    depth = np.where(holes, 0.0, fb.depth).astype(np.float32)
    valid = fb.valid_mask & ~holes
    d["inpaint_in"], d["inpaint_valid"] = depth.astype(np.float64), valid
    d["inpaint_out"] = inpaint_depth(depth.astype(np.float64), valid)
    d["inpaint_out_short"] = inpaint_depth(depth.astype(np.float64), valid, max_iters=7)
    ri = ref_intr(GEO, intr)
    ident = GEO.Pose.identity()
    tpose = GEO.Pose(truth.rotation, truth.translation)
    map_a = ref_map(G, GEO, params, ri, ident, 0)
    fr_a = RgbdFrame(color=fa.color, depth=fa.depth, valid_mask=fa.valid_mask, intrinsics=ri,
                     timestamp=0.0, index=0)
    fr_b = RgbdFrame(color=fb.color, depth=depth, valid_mask=valid, intrinsics=ri,
                     timestamp=1.0, index=1)
    d["base_depth"] = M.assemble_base_depth(fr_b, tpose, [map_a])
    d["target_depth"], d["target_valid"] = depth, valid
    cfg = M.MapperConfig(mapping_iters=4)
    gmap, losses = M.map_frame(fr_b, tpose, [(fr_a, ident, map_a)], cfg, seed=0)
    d["mf_losses"] = np.array(losses)
    for k in ("base_depth", "delta", "log_radius", "opacity_logit", "color", "active_mask"):
        d[f"mf_{k}"] = getattr(gmap, k)
    with _tf.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "m.bin")
        G.save_gaussian_map(path, gmap)
        d["mapfile"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8).copy()
    return d


BENCH_VIEWS = {"c3": 3, "c4": 5}


def golden_bench(cfg_name, state, ref_path):
    """One target view of a benched window (C3 640x480 / C4 1200x680, 8
    keyframes, the bench's init_params or the teacher-forced state
    helpers.forced_params) through the REAL reference (oracle/refwindow.py:
    its _prepare / _build_tile_lists / _forward_kernel / _backward_kernel,
    loss upstream and chain rule, all maps learnable -- delta D1), stored as
    compact exact digests: tile offsets and per-tile list hashes, loss terms,
    sampled pixels and Gaussians, per-frame gradient sums."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import time
    from helpers import forced_params, sample_indices, tile_digest
    from oracle import refwindow as RW
    from paper_2603_21055_b200 import scenes
    ref = RW.import_reference(ref_path)
    wc = scenes.config_c3() if cfg_name == "c3" else scenes.config_c4()
    params = wc.params if state == "init" else forced_params(wc.params)
    v = BENCH_VIEWS[cfg_name]
    ri, maps = RW.ref_maps(ref, wc.intr, wc.poses, params)
    fr = wc.frames[v]
    t0 = time.time()
    r = RW.window_view(ref, maps, wc.poses[v], ri, fr.color, fr.depth, fr.valid_mask,
                       keep_lists=True)
    print(f"{cfg_name}/{state}: reference view {v} in {time.time() - t0:.1f} s", flush=True)
    h, w = ri.height, ri.width
    ent = r.lists
    d = {"view": np.array(v), "n_surv": np.array(len(r.frame)),
         "offsets": np.asarray(r.offsets, dtype=np.int64),
         "tile_hash": tile_digest(r.offsets, r.frame[ent], r.pixel[ent]),
         "loss": np.array([r.color_l1, r.depth_l1])}
    px = sample_indices(h * w, 8000, 5)
    d["px"] = px
    d["px_color"] = r.color.reshape(-1, 3)[px]
    d["px_depth"] = r.depth.reshape(-1)[px]
    d["px_alpha"] = r.alpha.reshape(-1)[px]
    d["px_count"] = r.count.reshape(-1)[px]
    d["img_sums"] = np.array([r.color.sum(), r.depth.sum(), r.alpha.sum(), r.count.sum()])
    n_g = len(maps) * h * w
    gs = sample_indices(n_g, 20000, 6)
    d["gs"] = gs
    planes = np.zeros((len(maps), 6, h * w))
    for f, m in enumerate(maps):
        gc, gr, gl, gd = r.grads[m.frame_index]
        planes[f] = np.stack([gd.reshape(-1), gr.reshape(-1), gl.reshape(-1),
                              *gc.reshape(-1, 3).T])
    flat = planes.transpose(0, 2, 1).reshape(n_g, 6)
    d["g_sample"] = flat[gs]
    d["g_frame_sums"] = planes.sum(axis=2)
    d["g_frame_abs"] = np.abs(planes).sum(axis=2)
    return d


def main():
    sys.path.insert(0, ROOT)
    want = set(sys.argv[1:]) or {"c1", "window", "eig", "track", "ssim", "render_init", "voxels",
                                    "frame_driver", "bench"}
    tmp, G, GEO, M, R, T, RgbdFrame = import_reference()
    for cfg_name in ("c3", "c4"):
        for state in ("init", "forced"):
            if f"bench_{cfg_name}_{state}" in want or f"bench_{cfg_name}" in want or "bench" in want:
                np.savez_compressed(os.path.join(HERE, f"bench_{cfg_name}_{state}.npz"),
                                    **golden_bench(cfg_name, state, tmp))
    try:
        if "c1" in want:
            np.savez_compressed(os.path.join(HERE, "c1.npz"), **golden_c1(G, GEO, M, R, RgbdFrame))
        if "window" in want:
            np.savez_compressed(os.path.join(HERE, "window.npz"), **golden_window(G, GEO, R))
        if "eig" in want:
            np.savez_compressed(os.path.join(HERE, "eig.npz"), **golden_eig(GEO))
        if "track" in want:
            np.savez_compressed(os.path.join(HERE, "track.npz"), **golden_track(T, GEO))
        if "frame_driver" in want:
            np.savez_compressed(os.path.join(HERE, "frame_driver.npz"),
                                **golden_frame_driver(G, GEO, M, RgbdFrame))
        if "voxels" in want:
            np.savez_compressed(os.path.join(HERE, "voxels.npz"), **golden_voxels(T))
        if "render_init" in want:
            np.savez_compressed(os.path.join(HERE, "render_init.npz"),
                                **golden_render_init(G, GEO, T, RgbdFrame))
        if "ssim" in want:
            np.savez_compressed(os.path.join(HERE, "ssim.npz"),
                                **golden_ssim(M, G, GEO, R, RgbdFrame))
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
