"""Differentiable splatting of pixel-Gaussian maps -- drop-in for
/root/reference/pkg/src/raysplat/rasterizer.py.

``splat`` (rasterizer.py:366-392) and ``splat_backward`` (:395-484) keep the
reference signatures, argument meanings and error behaviour; inputs and
outputs are CUDA tensors (numpy inputs are accepted and uploaded).  Every
call runs the sm_100a kernels of libsgad.so (K1 project, K2 depth sort, K3
tile binning, K4 composite, K5 backward + chain); there is no CPU path.

Delta D1 (window mapping): ``learnable_map`` also accepts a sequence of map
positions or ``"all"``; the backward then returns one MapGradients per
learnable map.  A single all-learnable sweep followed by the per-map chain
is exactly what the reference computes with one ``splat_backward`` call per
map.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .geometry import Intrinsics, Pose, relative_pose

ALPHA_MAX = 0.999
TRANSMITTANCE_MIN = 1e-4
Z_NEAR = 1e-6
TILE = 16


@dataclass
class RenderOutput:
    """Composited target view (rasterizer.py:34-45); fp64 CUDA tensors."""

    color: torch.Tensor
    depth: torch.Tensor
    alpha: torch.Tensor
    contributors: torch.Tensor

    @property
    def shape(self):
        return tuple(self.depth.shape)


@dataclass
class MapGradients:
    """Gradients of one learnable map (rasterizer.py:48-55), zero where culled."""

    color: torch.Tensor
    radius: torch.Tensor
    opacity_logit: torch.Tensor
    delta: torch.Tensor


class Raster:
    """One sgad_raster handle: per-view device scratch for prepare/forward/backward."""

    def __init__(self, device=None):
        N.load()
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            N.check(N.load().sgad_raster_create(ctypes.byref(h)))
        self.h = h
        self.n_surv = 0
        self.n_pairs = 0
        self._frames = None
        self._keep = []

    def __del__(self):
        try:
            if self.h:
                N.load(require_cuda=False).sgad_raster_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def prepare(self, frames, cam, want_coef=False, stream=None):
        ns, npairs = ctypes.c_int64(), ctypes.c_int64()
        self._frames = frames
        N.check(N.load().sgad_raster_prepare(self.h, frames, len(frames), ctypes.byref(cam),
                                             int(want_coef), N.stream_ptr(stream),
                                             ctypes.byref(ns), ctypes.byref(npairs)))
        self.cam = cam
        self.n_surv, self.n_pairs = ns.value, npairs.value
        return self.n_surv, self.n_pairs

    def prepare_async(self, frames, cam, want_coef=False, counts=None, overflow=None, stream=None,
                      frames_dev=None):
        """The preparation without host synchronisation: ``counts`` (device
        int32[2], optional) receives (survivors, pairs); ``overflow`` (device
        int32[1], optional) is set to 1 if the view has more tile pairs than
        the reserved capacity (its results are then invalid); ``frames_dev``
        (optional device tensor holding ``frames``' bytes) is used instead of
        uploading the frame table (CUDA-graph capture)."""
        self._frames = frames
        N.check(N.load().sgad_raster_prepare_async(self.h, frames, len(frames), ctypes.byref(cam),
                                                   int(want_coef), N.ptr(frames_dev),
                                                   N.ptr(counts), N.ptr(overflow),
                                                   N.stream_ptr(stream)))
        self.cam = cam
        self.n_surv = self.n_pairs = -1

    def reserve(self, pair_capacity: int):
        N.check(N.load().sgad_raster_reserve(self.h, int(pair_capacity)))

    def forward(self, color=None, depth=None, alpha=None, count=None, save_state=False,
                target=None, stream=None):
        tgt = ctypes.byref(target) if target is not None else None
        N.check(N.load().sgad_raster_forward(self.h, N.ptr(color), N.ptr(depth), N.ptr(alpha),
                                             N.ptr(count), int(save_state), tgt,
                                             N.stream_ptr(stream)))

    def backward_exact(self, g_color, g_depth, g_alpha, map_grads, stream=None):
        arr = (ctypes.c_void_p * max(len(map_grads), 1))(*[N.ptr(t) for t in map_grads])
        N.check(N.load().sgad_raster_backward(self.h, 0, N.ptr(g_color), N.ptr(g_depth),
                                              N.ptr(g_alpha), arr, None, N.stream_ptr(stream)))

    def backward_fused(self, grad_accum, g_color=None, stream=None):
        """Fused backward into ``grad_accum``; ``g_color`` (device fp64
        [H, W, 3]) overrides the colour upstream (the tau != 0 objective)."""
        N.check(N.load().sgad_raster_backward(self.h, 1, N.ptr(g_color), None, None, None,
                                              N.ptr(grad_accum), N.stream_ptr(stream)))

    def forward_backward(self, target, grad_accum, stream=None):
        """Forward + fused L1 loss + fused backward in one kernel (tau = 0)."""
        N.check(N.load().sgad_raster_forward_backward(self.h, ctypes.byref(target),
                                                      N.ptr(grad_accum), N.stream_ptr(stream)))

    def survivors(self):
        n = self.n_surv
        dev = self.device
        out = {"gid": torch.empty(n, dtype=torch.int64, device=dev)}
        for k in ("u0", "v0", "z", "sigma", "opacity"):
            out[k] = torch.empty(n, dtype=torch.float64, device=dev)
        N.check(N.load().sgad_raster_get_survivors(
            self.h, N.ptr(out["gid"]), N.ptr(out["u0"]), N.ptr(out["v0"]), N.ptr(out["z"]),
            N.ptr(out["sigma"]), N.ptr(out["opacity"]), N.stream_ptr()))
        return out

    def tiles(self):
        nt = ctypes.c_int64()
        N.check(N.load().sgad_raster_tile_count(self.h, ctypes.byref(nt)))
        ranges = torch.empty((nt.value, 2), dtype=torch.int64, device=self.device)
        lists = torch.empty(max(self.n_pairs, 1), dtype=torch.int64, device=self.device)
        N.check(N.load().sgad_raster_get_tiles(self.h, N.ptr(ranges), N.ptr(lists),
                                               N.stream_ptr()))
        return ranges, lists[: self.n_pairs]


_tls = threading.local()


def get_raster(device=None) -> Raster:
    """Per-thread, per-device handle (the reference's kernels are re-entrant and
    called from pool threads, raysplat/pipeline.py:212)."""
    dev = torch.cuda.current_device() if device is None else torch.device(device).index
    cache = getattr(_tls, "rasters", None)
    if cache is None:
        cache = _tls.rasters = {}
    if dev not in cache:
        cache[dev] = Raster(torch.device("cuda", dev))
    return cache[dev]


def camera_of(intr: Intrinsics) -> N.Camera:
    return N.Camera(float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy),
                    int(intr.width), int(intr.height))


def learnable_set(learnable, n_maps) -> set:
    if learnable is None:
        return set()
    if isinstance(learnable, str):
        if learnable != "all":
            raise ValueError("learnable_map must be an int, a sequence of ints or 'all'")
        return set(range(n_maps))
    if isinstance(learnable, (int, np.integer)):
        if not -n_maps <= int(learnable) < n_maps:
            raise IndexError("learnable_map out of range")
        return {int(learnable) % n_maps}
    return {int(i) for i in learnable}


def frame_order(maps):
    """Emission order: by reference frame index, stable in map order."""
    return sorted(range(len(maps)), key=lambda i: maps[i].frame_index)


def build_frames(maps, target_pose: Pose, learn: set, order=None):
    """sgad_frame descriptors for one target view (relative poses on the host,
    evaluated with the reference's own expression, rasterizer.py:94)."""
    order = frame_order(maps) if order is None else order
    arr = (N.Frame * max(len(order), 1))()
    off = 0
    offsets = {}
    for pos, i in enumerate(order):
        m = maps[i]
        h, w = m.shape
        rel = relative_pose(target_pose, m.pose)
        fr = arr[pos]
        fr.planes = m.planes.data_ptr()
        fr.mask = m.mask_u8.data_ptr()
        fr.gauss_offset = off
        fr.frame_index = int(m.frame_index)
        fr.height, fr.width = int(h), int(w)
        fr.learnable = 1 if i in learn else 0
        fr.planes_f64 = 1 if m.planes.dtype == torch.float64 else 0
        si = m.intrinsics
        fr.fx, fr.fy, fr.cx, fr.cy = float(si.fx), float(si.fy), float(si.cx), float(si.cy)
        fr.rot[:] = [float(x) for x in np.asarray(rel.rotation).reshape(9)]
        fr.trans[:] = [float(x) for x in np.asarray(rel.translation).reshape(3)]
        offsets[i] = off
        off += int(h) * int(w)
    return arr, order, offsets, off


def _to_dev(x, dtype, device, shape=None):
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x))
    t = t.to(device=device, dtype=dtype).contiguous()
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"expected shape {tuple(shape)}, got {tuple(t.shape)}")
    return t


def _device_of(maps, device=None):
    if device is not None:
        return torch.device(device)
    for m in maps:
        return m.planes.device
    return torch.device("cuda", torch.cuda.current_device())


def splat(maps, target_pose: Pose, intrinsics: Intrinsics, normalize_depth: bool = False,
          device=None) -> RenderOutput:
    """Render source maps into the target camera (rasterizer.py:366-392).

    Independent of the order of ``maps``; an empty source set gives zeros."""
    maps = list(maps)
    dev = _device_of(maps, device)
    h, w = int(intrinsics.height), int(intrinsics.width)
    out = RenderOutput(torch.zeros((h, w, 3), dtype=torch.float64, device=dev),
                       torch.zeros((h, w), dtype=torch.float64, device=dev),
                       torch.zeros((h, w), dtype=torch.float64, device=dev),
                       torch.zeros((h, w), dtype=torch.int32, device=dev))
    if maps:
        with torch.cuda.device(dev):
            r = get_raster()
            frames, _, _, _ = build_frames(maps, target_pose, set())
            ns, _ = r.prepare(frames, camera_of(intrinsics))
            if ns:
                r.forward(out.color, out.depth, out.alpha, out.contributors)
    if normalize_depth:
        out.depth = torch.where(out.alpha > 1e-8, out.depth / torch.clamp(out.alpha, min=1e-8),
                                torch.zeros_like(out.depth))
    return out


def splat_backward(maps, target_pose: Pose, intrinsics: Intrinsics, grad_color, grad_depth,
                   grad_alpha, learnable_map=0, normalize_depth: bool = False, device=None):
    """Backpropagate image-space gradients into the learnable map(s)
    (rasterizer.py:395-484).  Gradients are fp64; culled Gaussians get zero."""
    maps = list(maps)
    learn = learnable_set(learnable_map, len(maps))
    dev = _device_of(maps, device)
    h, w = int(intrinsics.height), int(intrinsics.width)
    grads = {}
    for i in sorted(learn):
        mh, mw = maps[i].shape
        grads[i] = torch.zeros((6, mh, mw), dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        gc = _to_dev(grad_color, torch.float64, dev, (h, w, 3))
        gd = _to_dev(grad_depth, torch.float64, dev, (h, w))
        ga = _to_dev(grad_alpha, torch.float64, dev, (h, w)).clone()
        r = get_raster()
        frames, order, _, _ = build_frames(maps, target_pose, learn)
        ns, _ = r.prepare(frames, camera_of(intrinsics))
        if ns:
            if normalize_depth:
                # fold d_hat = d / max(a, eps) into the upstream (rasterizer.py:427-433)
                dep = torch.empty((h, w), dtype=torch.float64, device=dev)
                alp = torch.empty((h, w), dtype=torch.float64, device=dev)
                r.forward(None, dep, alp, None, save_state=True)
                safe_a = torch.clamp(alp, min=1e-8)
                covered = alp > 1e-8
                zero = torch.zeros_like(gd)
                ga = ga + torch.where(covered, -gd * dep / safe_a**2, zero)
                gd = torch.where(covered, gd / safe_a, zero)
            else:
                r.forward(save_state=True)
            table = [grads.get(i) for i in order]
            r.backward_exact(gc, gd.contiguous(), ga.contiguous(), table)
    res = {}
    for i, g in grads.items():
        res[i] = MapGradients(color=g[3:6].permute(1, 2, 0), radius=g[1], opacity_logit=g[2],
                              delta=g[0])
    if isinstance(learnable_map, (int, np.integer)):
        return res[int(learnable_map) % len(maps)]
    return [res[i] for i in sorted(learn)]


def inspect_view(maps, target_pose: Pose, intrinsics: Intrinsics):
    """Survivors (sorted order) and tile lists/ranges of one view -- the exact
    index data the reference keeps in _SplatBatch / _build_tile_lists, for
    bit-exact parity tests.  Returns numpy arrays plus (map position, pixel)
    of every survivor."""
    maps = list(maps)
    r = get_raster(_device_of(maps))
    frames, order, offsets, _ = build_frames(maps, target_pose, set())
    r.prepare(frames, camera_of(intrinsics))
    s = {k: v.cpu().numpy() for k, v in r.survivors().items()}
    ranges, lists = r.tiles()
    starts = np.array([offsets[i] for i in order], dtype=np.int64)
    pos = np.searchsorted(starts, s["gid"], side="right") - 1
    s["map_pos"] = np.array(order, dtype=np.int64)[pos] if len(pos) else pos
    s["pixel"] = s["gid"] - starts[pos] if len(pos) else s["gid"]
    return s, ranges.cpu().numpy(), lists.cpu().numpy()
