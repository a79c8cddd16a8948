"""Window iteration driven through the REAL reference -- test and baseline
infrastructure, never the product.

Runs the reference package ``raysplat`` itself (the copy installed under
``baseline/_ref`` -- it travels to the GPU box -- or any directory holding a
copy of ``/root/reference/pkg/src``) through its own internals, as
BASELINE.md section 2 prescribes for the window configurations (delta D1: all
maps learnable, every view rendered):

* ``_prepare`` with every survivor learnable (rasterizer.py:79-175), its
  ``_build_tile_lists`` (:178-218), ``_forward_kernel`` (:221-269) and
  ``_backward_kernel`` (:272-363) -- unmodified Numba kernels;
* the loss upstream of ``mapping_loss`` (mapper.py:118-152, tau = 0) and the
  chain rule of ``splat_backward`` (rasterizer.py:462-483), restated once for
  all survivors and scattered per source map;
* ``MapOptimizer.step`` (mapper.py:73-95), the reference's own Adam.

A one-sweep all-learnable backward followed by the per-map chain is
bit-identical to one ``splat_backward`` call per map.  The
survivor -> frame map is not kept in ``_SplatBatch``; it is read from the
keys handed to ``np.lexsort`` (rasterizer.py:157-158) through a thread-local
spy on the module's ``np`` (the reference's kernels are ``nogil``; views run
in a thread pool like raysplat/pipeline.py:212).

Only ``tests/``, ``tests/golden/make_golden.py`` and bench.py's CPU legs
(``bench_cpu.py``) use this module.
"""

from __future__ import annotations

import os
import sys
import threading
from dataclasses import dataclass
from types import SimpleNamespace

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASELINE_REF = os.path.join(ROOT, "baseline", "_ref")

_tls = threading.local()


def _lexsort_spy(keys, axis=-1):
    """np.lexsort that also records the sorted frame key of the calling
    thread's last ``_prepare`` (rasterizer.py:157: keys = pixel, frame, z)."""
    order = np.lexsort(keys, axis=axis)
    if len(keys) == 3:
        _tls.frame = np.asarray(keys[1])[order]
    return order


def _numpy_spy():
    """A module object with numpy's namespace and the recording lexsort (a
    real module, so the reference's Numba kernels still resolve ``np.*``)."""
    import types
    mod = types.ModuleType("numpy")
    mod.__dict__.update(np.__dict__)
    mod.lexsort = _lexsort_spy
    mod._sgad_spy = True
    return mod


def import_reference(path: str | None = None):
    """Import raysplat from ``path`` (default ``baseline/_ref``); returns a
    namespace of its modules with the lexsort spy installed."""
    path = path or BASELINE_REF
    if not os.path.isdir(os.path.join(path, "raysplat")):
        raise FileNotFoundError(f"no raysplat package under {path} (see DESIGN.md: "
                                "pip install --target baseline/_ref)")
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", f"sgad_numba_{os.getuid()}"))
    sys.dont_write_bytecode = True
    if path not in sys.path:
        sys.path.insert(0, path)
    import raysplat.gaussians as G
    import raysplat.geometry as GEO
    import raysplat.mapper as M
    import raysplat.rasterizer as R
    if not getattr(R.np, "_sgad_spy", False):
        R.np = _numpy_spy()
    return SimpleNamespace(G=G, GEO=GEO, M=M, R=R, path=path)


def ref_maps(ref, intr, poses, params):
    """Reference PixelGaussianMaps (fp64 copies) of a window."""
    ri = ref.GEO.Intrinsics(fx=intr.fx, fy=intr.fy, cx=intr.cx, cy=intr.cy, width=intr.width,
                            height=intr.height)
    maps = []
    for i, p in enumerate(params):
        pose = ref.GEO.Pose(np.asarray(poses[i].rotation, np.float64),
                            np.asarray(poses[i].translation, np.float64))
        maps.append(ref.G.PixelGaussianMap(
            frame_index=i, pose=pose, intrinsics=ri,
            base_depth=np.array(p.base_depth, np.float64), delta=np.array(p.delta, np.float64),
            color=np.array(p.color, np.float64), log_radius=np.array(p.log_radius, np.float64),
            opacity_logit=np.array(p.opacity_logit, np.float64),
            active_mask=np.array(p.active_mask, bool)))
    return ri, maps


@dataclass
class ViewResult:
    color_l1: float
    depth_l1: float
    color: np.ndarray
    depth: np.ndarray
    alpha: np.ndarray
    count: np.ndarray
    grads: dict          # frame_index -> (g_color [h,w,3], g_radius, g_logit, g_delta)
    offsets: np.ndarray | None = None
    lists: np.ndarray | None = None
    frame: np.ndarray | None = None     # survivor frame, depth order
    pixel: np.ndarray | None = None     # survivor pixel, depth order


def window_view(ref, maps, pose, intr, tcolor, tdepth, tmask, rho=0.8, sigma=1.0,
                keep_lists=False) -> ViewResult:
    """One target view of a window iteration (tau = 0, un-normalised depth)."""
    R = ref.R
    h, w = intr.height, intr.width
    tpose = ref.GEO.Pose(np.asarray(pose.rotation, np.float64),
                         np.asarray(pose.translation, np.float64))
    _tls.frame = None
    batch = R._prepare(maps, tpose, intr, learnable_map=-1)
    n = len(batch.z)
    frame = _tls.frame if n else np.zeros(0, np.int64)
    batch.learnable[:] = 1
    color = np.zeros((h, w, 3))
    depth = np.zeros((h, w))
    alpha = np.zeros((h, w))
    count = np.zeros((h, w), dtype=np.int32)
    offsets = lists = None
    if n:
        offsets, lists = R._build_tile_lists(batch.u0, batch.v0, batch.sigma, h, w, R._TILE)
        R._forward_kernel(batch.u0, batch.v0, batch.z, batch.sigma, batch.opacity, batch.color,
                          offsets, lists, h, w, R._TILE, color, depth, alpha, count)
    # mapper.py:118-152 (tau = 0)
    tc = np.asarray(tcolor, dtype=np.float64)
    n_color = color.size
    resid = color - tc
    color_l1 = float(np.abs(resid).sum() / n_color)
    mask = np.asarray(tmask, dtype=bool)
    n_depth = int(mask.sum())
    dres = depth - np.asarray(tdepth, dtype=np.float64)
    depth_l1 = float(np.abs(dres[mask]).sum() / n_depth) if n_depth else 0.0
    g_color = np.ascontiguousarray(rho * np.sign(resid) / n_color)
    g_depth = np.ascontiguousarray(sigma * np.sign(dres) * mask / n_depth if n_depth
                                   else np.zeros_like(dres))
    g_alpha = np.zeros_like(g_depth)
    grads = {}
    for m in maps:
        mh, mw = m.shape
        grads[m.frame_index] = (np.zeros((mh, mw, 3)), np.zeros((mh, mw)), np.zeros((mh, mw)),
                                np.zeros((mh, mw)))
    if n:
        gc = np.zeros((n, 3))
        gop, gu, gv, gs, gz = (np.zeros(n) for _ in range(5))
        R._backward_kernel(batch.u0, batch.v0, batch.z, batch.sigma, batch.opacity, batch.color,
                           batch.learnable, offsets, lists, h, w, R._TILE, g_color, g_depth,
                           g_alpha, gc, gop, gu, gv, gs, gz)
        # rasterizer.py:462-483 for every survivor, scattered to its map
        y, z, dir_t = batch.y, batch.z, batch.dir_t
        g_radius = gs * batch.fx / z
        g_z_total = (gz - gs * batch.sigma / z - gu * batch.fx * y[:, 0] / z**2
                     - gv * batch.fy * y[:, 1] / z**2)
        g_y0 = gu * batch.fx / z
        g_y1 = gv * batch.fy / z
        g_dadj = g_y0 * dir_t[:, 0] + g_y1 * dir_t[:, 1] + g_z_total * dir_t[:, 2]
        g_logit = gop * batch.opacity * (1.0 - batch.opacity)
        for m in maps:
            sel = frame == m.frame_index
            if not sel.any():
                continue
            pix = batch.pixel_index[sel]
            base = m.base_depth.reshape(-1)[pix]
            delta = m.delta.reshape(-1)[pix]
            sgn = np.where(base + delta >= 0.0, 1.0, -1.0)
            o_c, o_r, o_l, o_d = grads[m.frame_index]
            o_c.reshape(-1, 3)[pix] = gc[sel]
            o_r.reshape(-1)[pix] = g_radius[sel]
            o_l.reshape(-1)[pix] = g_logit[sel]
            o_d.reshape(-1)[pix] = g_dadj[sel] * sgn
    res = ViewResult(color_l1, depth_l1, color, depth, alpha, count, grads)
    if keep_lists:
        res.offsets, res.lists = offsets, lists
        res.frame, res.pixel = frame, batch.pixel_index
    return res


class WindowStep:
    """A (bounded) window iteration on the reference: ``views`` rendered in a
    thread pool (raysplat/pipeline.py:212), gradients summed per map, then the
    reference's ``MapOptimizer.step`` on every map."""

    def __init__(self, ref, intr, poses, params, frames, cfg=None):
        self.ref = ref
        self.ri, self.maps = ref_maps(ref, intr, poses, params)
        self.poses = poses
        self.frames = frames
        self.cfg = cfg or ref.M.MapperConfig(tau=0.0)
        self.opts = [ref.M.MapOptimizer(m, self.cfg) for m in self.maps]

    def step(self, views, pool=None):
        def one(v):
            fr = self.frames[v]
            return window_view(self.ref, self.maps, self.poses[v], self.ri, fr.color, fr.depth,
                               fr.valid_mask, self.cfg.rho, self.cfg.sigma)
        results = list(pool.map(one, views)) if pool is not None else [one(v) for v in views]
        total = 0.0
        for r in results:
            total += self.cfg.rho * r.color_l1 + self.cfg.sigma * r.depth_l1
        for m, opt in zip(self.maps, self.opts):
            acc = None
            for r in results:
                g = r.grads[m.frame_index]
                acc = [a.copy() for a in g] if acc is None else [a + b for a, b in zip(acc, g)]
            opt.step(self.ref.R.MapGradients(color=acc[0], radius=acc[1], opacity_logit=acc[2],
                                             delta=acc[3]))
        return total
