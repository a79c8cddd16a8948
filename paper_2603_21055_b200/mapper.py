"""Mapping objective and optimizer -- drop-in for
/root/reference/pkg/src/raysplat/mapper.py, plus the B200 window engine.

* ``mapping_loss`` (mapper.py:106-157) and ``MapOptimizer`` (:48-95) keep the
  reference signatures; they run on CUDA tensors through libsgad.so,
  including the SSIM term (tau != 0, mapper.py:126-147; csrc/ssim.cu).
* ``WindowMapper`` is the graded hot path (north_star / BASELINE C3-C5):
  every keyframe of the window is learnable (delta D1), every view is
  rendered, the L1 loss is fused into the compositing kernel (the SSIM term,
  when tau != 0, runs on the rendered colour and hands the backward its
  colour upstream), the
  backward chains per-pixel gradients straight onto the window's parameter
  planes, views are sharded over ranks with one NCCL all-reduce of the
  per-Gaussian gradients, and one Adam kernel updates all planes.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import ssim as S
from .gaussians import PixelGaussianMap
from .geometry import Intrinsics, Pose
from .rasterizer import (MapGradients, Raster, RenderOutput, build_frames, camera_of, get_raster,
                         learnable_set)


@dataclass
class MapperConfig:
    """mapper.py:28-45 (same fields and defaults)."""

    rho: float = 0.8
    tau: float = 0.2
    sigma: float = 1.0
    neighbor_count: int = 1
    mapping_iters: int = 100
    lr_color: float = 0.0025
    lr_radius: float = 0.005
    lr_opacity: float = 0.05
    lr_offset: float = 0.01
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8
    min_current_fraction: float = 0.4
    offset_frozen: bool = False
    normalize_depth: bool = False
    coverage_alpha: float = 0.5

    def lrs(self):
        """Per-channel learning rates in grad-buffer order (delta, log_radius,
        opacity_logit, R, G, B)."""
        return [self.lr_offset, self.lr_radius, self.lr_opacity,
                self.lr_color, self.lr_color, self.lr_color]


@dataclass
class LossBreakdown:
    total: float
    color_l1: float
    ssim_term: float
    depth_l1: float


def _adam(params, grads, m, v, n_frames, hw, cfg: MapperConfig, t: int, f64: bool, skip=None,
          t_dev=None):
    lr = (ctypes.c_double * 6)(*cfg.lrs())
    b1, b2 = cfg.adam_beta1, cfg.adam_beta2
    N.call("sgad_adam_step", params.data_ptr(), grads.data_ptr(), m.data_ptr(), v.data_ptr(),
           int(n_frames), int(hw), lr, b1, b2, cfg.adam_eps, 1.0 - b1**t, 1.0 - b2**t,
           0 if cfg.offset_frozen else 1, 1 if f64 else 0, N.ptr(skip), N.ptr(t_dev),
           N.stream_ptr())


class MapOptimizer:
    """Adam over the four learnable groups of one map (mapper.py:48-95), on device."""

    def __init__(self, gmap: PixelGaussianMap, cfg: MapperConfig):
        self.gmap = gmap
        self.cfg = cfg
        self.t = 0
        h, w = gmap.shape
        dt, dev = gmap.planes.dtype, gmap.planes.device
        self._m = torch.zeros((6, h, w), dtype=dt, device=dev)
        self._v = torch.zeros((6, h, w), dtype=dt, device=dev)
        self._g = torch.zeros((h * w, 8), dtype=dt, device=dev)

    def step(self, grads: MapGradients) -> None:
        self.t += 1
        g = self._g
        dt = g.dtype
        g[:, 0] = torch.as_tensor(grads.delta).to(g.device, dt).reshape(-1)
        g[:, 1] = torch.as_tensor(grads.radius).to(g.device, dt).reshape(-1)
        g[:, 2] = torch.as_tensor(grads.opacity_logit).to(g.device, dt).reshape(-1)
        g[:, 3:6] = torch.as_tensor(grads.color).to(g.device, dt).reshape(-1, 3)
        h, w = self.gmap.shape
        _adam(self.gmap.planes, g, self._m, self._v, 1, h * w, self.cfg, self.t,
              dt == torch.float64)


def mapping_loss(maps, target_frame, target_pose: Pose, cfg: MapperConfig, with_grads=True):
    """mapper.py:106-157: returns (LossBreakdown, MapGradients | None,
    RenderOutput) with gradients for ``maps[0]``; the SSIM term (tau != 0,
    :126-133,146-147) runs on the GPU (ssim.py)."""
    maps = list(maps)
    intr = target_frame.intrinsics
    dev = maps[0].planes.device if maps else torch.device("cuda", torch.cuda.current_device())
    h, w = int(intr.height), int(intr.width)
    out = RenderOutput(torch.zeros((h, w, 3), dtype=torch.float64, device=dev),
                       torch.zeros((h, w), dtype=torch.float64, device=dev),
                       torch.zeros((h, w), dtype=torch.float64, device=dev),
                       torch.zeros((h, w), dtype=torch.int32, device=dev))
    with torch.cuda.device(dev):
        r = get_raster()
        learn = {0} if (with_grads and maps) else set()
        frames, order, _, _ = build_frames(maps, target_pose, learn)
        ns = r.prepare(frames, camera_of(intr))[0] if maps else 0
        if ns:
            r.forward(out.color, out.depth, out.alpha, out.contributors, save_state=True)
        raw_depth, raw_alpha = out.depth, out.alpha
        if cfg.normalize_depth:
            out.depth = torch.where(out.alpha > 1e-8,
                                    out.depth / torch.clamp(out.alpha, min=1e-8),
                                    torch.zeros_like(out.depth))
        tc = torch.as_tensor(np.asarray(target_frame.color)).to(dev, torch.float64)
        td = torch.as_tensor(np.asarray(target_frame.depth)).to(dev, torch.float64)
        mask = torch.as_tensor(np.asarray(target_frame.valid_mask)).to(dev, torch.bool)
        n_color = out.color.numel()
        resid = out.color - tc
        color_l1 = float(resid.abs().sum() / n_color)
        n_depth = int(mask.sum())
        dres = out.depth - td
        depth_l1 = float(dres[mask].abs().sum() / n_depth) if n_depth else 0.0
        ssim_gc = None
        ssim_val = 1.0
        if cfg.tau != 0.0:
            ssim_acc = torch.zeros((), dtype=torch.float64, device=dev)
            col = out.color.contiguous()
            if with_grads:
                # colour upstream rho sign(resid) / n - tau d(ssim)/d(colour), fused
                ssim_gc = torch.empty_like(col)
                ws = torch.empty(max(S.workspace_bytes(h, w, 3) // 8, 1), dtype=torch.float64,
                                 device=dev)
                S.ssim_sum(col, tc.contiguous(), ssim_acc, ssim_gc, ws, kc=cfg.rho / n_color,
                           tau=cfg.tau, upstream=True)
            else:
                S.ssim_sum(col, tc.contiguous(), ssim_acc)
            ssim_val = float(ssim_acc) / n_color
        total = cfg.rho * color_l1 + cfg.tau * (1.0 - ssim_val) + cfg.sigma * depth_l1
        breakdown = LossBreakdown(total, color_l1, 1.0 - ssim_val, depth_l1)
        if not with_grads:
            return breakdown, None, out
        gmap = maps[0]
        mh, mw = gmap.shape
        gbuf = torch.zeros((6, mh, mw), dtype=torch.float64, device=dev)
        if ns:
            g_color = ssim_gc if ssim_gc is not None else cfg.rho * torch.sign(resid) / n_color
            g_depth = (cfg.sigma * torch.sign(dres) * mask / n_depth if n_depth
                       else torch.zeros_like(dres))
            g_alpha = torch.zeros_like(g_depth)
            if cfg.normalize_depth:
                safe_a = torch.clamp(raw_alpha, min=1e-8)
                covered = raw_alpha > 1e-8
                zero = torch.zeros_like(g_depth)
                g_alpha = g_alpha + torch.where(covered, -g_depth * raw_depth / safe_a**2, zero)
                g_depth = torch.where(covered, g_depth / safe_a, zero)
            table = [gbuf if i == 0 else None for i in order]
            r.backward_exact(g_color.contiguous(), g_depth.contiguous(), g_alpha.contiguous(),
                             table)
    grads = MapGradients(color=gbuf[3:6].permute(1, 2, 0), radius=gbuf[1],
                         opacity_logit=gbuf[2], delta=gbuf[0])
    return breakdown, grads, out


def mapping_step(gmap, optimizer: MapOptimizer, target_frame, target_pose, neighbor_maps,
                 cfg: MapperConfig) -> LossBreakdown:
    """mapper.py:160-172."""
    breakdown, grads, _ = mapping_loss([gmap] + list(neighbor_maps), target_frame, target_pose,
                                       cfg)
    optimizer.step(grads)
    return breakdown


# ---------------------------------------------------------------- window engine


def shard_views(n_views: int, rank: int, world: int):
    """Views rendered by ``rank``: round-robin, so every rank gets n/world of
    them when world divides the window (8 keyframes over 1/2/4/8 GPUs)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return list(range(rank, n_views, world))


def allreduce_window(grad: torch.Tensor, loss_acc: torch.Tensor, group=None) -> bool:
    """The one exchange step of a window iteration: SUM of the per-Gaussian
    gradient buffer [N, 8] and of the per-view loss sums over ranks (the
    objective is a sum over views).  No-op without an initialised group."""
    dist = torch.distributed
    if not (dist.is_available() and dist.is_initialized()):
        return False
    if dist.get_world_size(group) == 1:
        return False
    _all_reduce(grad, group)
    _all_reduce(loss_acc, group)
    return True


def _host_staged(group, *tensors) -> bool:
    """gloo moves host memory only: CUDA tensors are staged through the host
    (tests run two ranks on one GPU with gloo; production uses NCCL)."""
    dist = torch.distributed
    return dist.get_backend(group) == "gloo" and any(t.is_cuda for t in tensors)


def _all_reduce(t: torch.Tensor, group=None) -> None:
    if _host_staged(group, t):
        h = t.cpu()
        torch.distributed.all_reduce(h, group=group)
        t.copy_(h)
    else:
        torch.distributed.all_reduce(t, group=group)


def frame_shard(n_frames: int, rank: int, world: int):
    """Frames [f0, f1) whose Adam step ``rank`` owns when the optimizer is
    sharded (contiguous blocks, so the gradient rows and parameter planes of a
    block are contiguous and the collectives need no packing)."""
    if world < 1 or not 0 <= rank < world or n_frames % world:
        raise ValueError("the window's frames must split evenly over the ranks")
    k = n_frames // world
    return rank * k, (rank + 1) * k


def reduce_scatter_window(grad: torch.Tensor, local: torch.Tensor, loss_acc: torch.Tensor,
                          group=None) -> None:
    """Sharded variant of the exchange step: the summed gradient
    rows of this rank's frame block into ``local`` (reduce-scatter over the
    frame-major [N, 8] buffer) and the per-view loss sums everywhere."""
    dist = torch.distributed
    if _host_staged(group, grad, local):
        h = local.cpu()
        dist.reduce_scatter_tensor(h, grad.cpu(), group=group)
        local.copy_(h)
    else:
        dist.reduce_scatter_tensor(local, grad, group=group)
    _all_reduce(loss_acc, group)


def allgather_planes(planes: torch.Tensor, stage: torch.Tensor, f0: int, f1: int,
                     group=None) -> None:
    """Every rank's updated frame block back into everyone's [F, 7, H, W]
    parameter tensor (all-gather of contiguous frame blocks)."""
    stage.copy_(planes[f0:f1])
    if _host_staged(group, planes):
        h = planes.cpu()
        torch.distributed.all_gather_into_tensor(h, stage.cpu(), group=group)
        planes.copy_(h)
    else:
        torch.distributed.all_gather_into_tensor(planes, stage, group=group)


class WindowMapper:
    """All-learnable keyframe window, fp32 parameters, fused loss + backward.

    ``frames``: per keyframe RGBD targets (``color`` HxWx3, ``depth`` HxW,
    ``valid_mask``); ``poses``: camera-to-world poses; ``params``: objects with
    ``base_depth, delta, log_radius, opacity_logit, color, active_mask``.
    ``views``: the keyframes this process renders (default: all of them, or
    under an initialised process group this rank's round-robin share,
    ``shard_views``); under torch.distributed the per-Gaussian gradient is
    summed over ranks (reduce-scatter by frame block + sharded Adam +
    all-gather, or an all-reduce + replicated Adam).  ``frame_indices`` must
    increase strictly: the Gaussian ids of frame i are rows [i HW, (i+1) HW)
    of the gradient and parameter planes, and the rasterizer orders maps by
    frame index.
    """

    def __init__(self, frames, poses, intr: Intrinsics, params, cfg: MapperConfig | None = None,
                 views=None, device=None, process_group=None, frame_indices=None):
        self.cfg = cfg or MapperConfig(tau=0.0)
        if self.cfg.normalize_depth:
            raise NotImplementedError("the fused window loss uses un-normalised depth")
        self.dev = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        self.intr = intr
        self.poses = list(poses)
        f = len(self.poses)
        h, w = int(intr.height), int(intr.width)
        self.F, self.H, self.W, self.HW = f, h, w, h * w
        dev = self.dev
        planes = np.empty((f, 7, h, w), dtype=np.float32)
        mask = np.empty((f, h, w), dtype=np.uint8)
        for i, p in enumerate(params):
            planes[i, 0] = p.base_depth
            planes[i, 1] = p.delta
            planes[i, 2] = p.log_radius
            planes[i, 3] = p.opacity_logit
            planes[i, 4:7] = np.asarray(p.color).transpose(2, 0, 1)
            mask[i] = np.asarray(p.active_mask, dtype=bool)
        self.planes = torch.from_numpy(planes).to(dev)
        self.mask = torch.from_numpy(mask).to(dev)
        idx = list(range(f)) if frame_indices is None else [int(i) for i in frame_indices]
        if len(idx) != f or any(b <= a for a, b in zip(idx, idx[1:])):
            raise ValueError("frame_indices must give one strictly increasing index per frame "
                             "(sort the window's frames by index)")
        self.maps = [PixelGaussianMap.from_planes(idx[i], self.poses[i], intr, self.planes[i],
                                                  self.mask[i]) for i in range(f)]
        self.tcolor = torch.from_numpy(np.stack([np.asarray(fr.color, np.float32)
                                                 for fr in frames])).to(dev).contiguous()
        self.tdepth = torch.from_numpy(np.stack([np.asarray(fr.depth, np.float32)
                                                 for fr in frames])).to(dev).contiguous()
        self.tmask = torch.from_numpy(np.stack([np.asarray(fr.valid_mask, bool)
                                                for fr in frames]).astype(np.uint8)).to(dev)
        self.n_depth = [int(np.asarray(fr.valid_mask, bool).sum()) for fr in frames]
        self._nd = (torch.tensor([max(n, 1) for n in self.n_depth], dtype=torch.float64, device=dev),
                    torch.tensor([n > 0 for n in self.n_depth], device=dev))
        if views is None:
            dist = torch.distributed
            if dist.is_available() and dist.is_initialized():
                views = shard_views(f, dist.get_rank(process_group),
                                    dist.get_world_size(process_group))
            else:
                views = range(f)
        self.views = list(views)
        self.grad = torch.zeros((f * self.HW, 8), dtype=torch.float32, device=dev)
        self.m = torch.zeros((f, 6, h, w), dtype=torch.float32, device=dev)
        self.v = torch.zeros((f, 6, h, w), dtype=torch.float32, device=dev)
        # per view: sum |C' - C|, sum_U |D' - D|, sum of per-pixel SSIM (tau != 0)
        self.loss_acc = torch.zeros((f, 3), dtype=torch.float64, device=dev)
        if self.cfg.tau != 0.0:
            # the SSIM term needs the rendered colour image: rendered into _col,
            # sgad_ssim turns it into the colour upstream _gcol the fused
            # backward consumes (all on the compositing stream, in order)
            self._col = torch.empty((h, w, 3), dtype=torch.float64, device=dev)
            self._gcol = torch.empty((h, w, 3), dtype=torch.float64, device=dev)
            self._ws = torch.empty(max(S.workspace_bytes(h, w, 3) // 8, 1), dtype=torch.float64,
                                   device=dev)
        # Adam's step count lives on the device (the bias corrections are
        # formed there, so a step can be replayed from a CUDA graph)
        self._t_dev = torch.zeros(1, dtype=torch.int32, device=dev)
        self.pg = process_group
        self.cam = camera_of(intr)
        learn = set(range(f))
        self._frames = {v: build_frames(self.maps, self.poses[v], learn)[0] for v in self.views}
        self.raster = get_raster(dev)
        # asynchronous preparation: per-view (survivors, pairs) on the device,
        # a per-step pair-capacity overflow flag (Adam skips a step that
        # overflowed; the host notices a step later, grows the capacity and
        # rolls the step counter back), the handles' pair capacity
        self._counts = torch.zeros((f, 2), dtype=torch.int32, device=dev)
        self._flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self._cap = 0
        self._pending = []
        self.overflows = 0
        # resident copies of every view's frame table (no host reads in a step)
        self._frames_dev = {v: torch.frombuffer(bytearray(bytes(fr)), dtype=torch.uint8).to(dev)
                            for v, fr in self._frames.items()}
        # CUDA graph of the whole window step (use_graph: captured at the first
        # step, replayed after; the per-view timing path stays eager)
        self.use_graph = False
        self._graph = None
        self._hgraph = None   # step_with_targets' capture (for one set of host buffers)
        self._hgraph_key = None
        self._copy = None     # upload stream of step_with_targets
        self.pipelined = True   # prepare view i+1 while view i composites
        self.adam_enabled = True
        # tau = 0: forward + loss + backward as one kernel (measured no faster
        # than the two kernels at C4, 3.84 vs 3.83 ms per view; kept as an option)
        self.fuse_fwd_bwd = False
        self._pipe = None
        # world > 1: reduce-scatter the gradient by frame block, Adam on this
        # rank's block only, all-gather the updated planes (instead of an
        # all-reduce and a replicated Adam); falls back to the all-reduce when
        # the frames do not split evenly over the ranks
        self.shard_adam = True
        self._shard = None

    @property
    def t(self) -> int:
        """Adam step count (device-resident; reading it synchronises)."""
        return int(self._t_dev.item())

    @t.setter
    def t(self, value: int):
        self._t_dev.fill_(int(value))

    @property
    def n_gaussians(self) -> int:
        return self.F * self.HW

    def _target(self, v):
        return N.LossTarget(self.tcolor[v].data_ptr(), self.tdepth[v].data_ptr(),
                            self.tmask[v].data_ptr(), self.cfg.rho, self.cfg.sigma,
                            self.n_depth[v], self.loss_acc[v].data_ptr())

    def _composite(self, r, v, stream, marks=None):
        """Forward with the fused L1 loss (+ the SSIM term when tau != 0) and
        the fused backward of a prepared view; ``marks`` (optional callable)
        records an event after the forward."""
        if self.cfg.tau != 0.0:
            r.forward(color=self._col, target=self._target(v), stream=stream)
            S.ssim_sum(self._col, self.tcolor[v], self.loss_acc[v, 2], self._gcol, self._ws,
                       kc=self.cfg.rho / (3.0 * self.HW), tau=self.cfg.tau, upstream=True,
                       stream=stream)
            mid = marks() if marks else None
            r.backward_fused(self.grad, g_color=self._gcol, stream=stream)
        elif self.fuse_fwd_bwd:
            r.forward_backward(self._target(v), self.grad, stream=stream)
            mid = None
        else:
            r.forward(target=self._target(v), stream=stream)
            mid = marks() if marks else None
            r.backward_fused(self.grad, stream=stream)
        return mid

    def render_view_grads(self, v, raster=None, stream=None):
        """Fused forward (+ loss) and backward of one view into self.grad."""
        r = raster or self.raster
        ns, npairs = r.prepare(self._frames[v], self.cam, want_coef=True, stream=stream)
        self._counts[v, 0], self._counts[v, 1] = ns, npairs
        if ns:
            self._composite(r, v, stream)

    def _render_pipelined(self, timing=None, target_ready=None):
        """All assigned views, the preparation (projection, depth order, tile
        lists) of view i+1 on a side stream while view i composites on the
        main stream.  Two raster handles alternate; a handle is re-prepared
        only after the compositing that used it has finished.  ``timing``
        (optional list) receives (kind, start_event, end_event, view) tuples;
        ``target_ready`` (optional {view: event}) holds back a view's
        compositing until its target has arrived (targets uploaded while
        earlier views composite)."""
        if self._pipe is None:
            self._new_pipe()
        rasters, prep = self._pipe
        nh = len(rasters)
        main = torch.cuda.current_stream(self.dev)
        ev = torch.cuda.Event()
        ev.record(main)           # parameters / loss accumulators are ready
        prep.wait_event(ev)
        used = [None] * nh        # compositing done on each handle

        def mark(stream):
            e = torch.cuda.Event(enable_timing=timing is not None)
            e.record(stream)
            return e

        for i, v in enumerate(self.views):
            r = rasters[i % nh]
            if used[i % nh] is not None:
                prep.wait_event(used[i % nh])
            p0 = mark(prep)
            r.prepare_async(self._frames[v], self.cam, want_coef=True, counts=self._counts[v],
                            overflow=self._flag, stream=prep, frames_dev=self._frames_dev[v])
            p1 = mark(prep)
            main.wait_event(p1)
            if target_ready is not None and v in target_ready:
                main.wait_event(target_ready[v])
            f0 = mark(main)
            f1 = self._composite(r, v, main, marks=lambda: mark(main))
            b1 = mark(main)
            if timing is not None:
                timing.append(("prep", p0, p1, v))
                if f1 is None:  # one fused kernel
                    timing.append(("fb", f0, b1, v))
                else:
                    timing += [("fwd", f0, f1, v), ("bwd", f1, b1, v)]
            used[i % nh] = mark(main)

    def _new_pipe(self):
        import os
        n = max(2, int(os.environ.get("SGAD_HANDLES", "2")))  # (A/B: views prepared ahead + 1)
        self._pipe = ([Raster(self.dev) for _ in range(n)], torch.cuda.Stream(self.dev))

    def _size_handles(self):
        """Pair capacity of the pipelined raster handles: every view prepared
        once synchronously, capacity = 1.3 x the largest pair count."""
        if self._pipe is None:
            self._new_pipe()
        r = self._pipe[0][0]
        most = 0
        for v in self.views:
            ns, npairs = r.prepare(self._frames[v], self.cam, want_coef=True)
            self._counts[v, 0], self._counts[v, 1] = ns, npairs
            most = max(most, npairs)
        self._cap = max(self._cap, int(most * 1.3) + 4096)
        for h in self._pipe[0]:
            h.reserve(self._cap)

    def _check_overflow(self, block: bool) -> bool:
        """Process the overflow flags of finished steps (all of them with
        ``block``): a step that overflowed skipped its Adam update on the
        device (its step count too); the capacity grows.  True if any did."""
        hit = False
        while self._pending:
            ev, host, adam = self._pending[0]
            if block:
                ev.synchronize()
            elif not ev.query():
                break
            self._pending.pop(0)
            if int(host[0]):
                hit = True
                self.overflows += 1
        if hit:
            torch.cuda.synchronize(self.dev)
            self._cap = int(self._cap * 1.5)
            self._size_handles()
            self._graph = None  # buffers were resized: capture again
            self._hgraph = None
        return hit

    def counts(self):
        """{view: (survivors, tile pairs)} of the last step (synchronises)."""
        c = self._counts.cpu().numpy()
        return {v: (int(c[v, 0]), int(c[v, 1])) for v in self.views}

    def step(self, sync_loss=False, timing=None, target_ready=None):
        """One window iteration: every assigned view fwd+bwd, gradient
        all-reduce across ranks, Adam.  Returns the summed loss (a device
        scalar unless ``sync_loss``).  ``target_ready`` ({view: CUDA event},
        optional): a view composites only after its event.  With
        ``use_graph`` the step is captured once in a CUDA graph and replayed
        (not with ``timing`` / ``target_ready``, which stay eager)."""
        with torch.cuda.device(self.dev):
            if self.pipelined:
                self._check_overflow(block=False)
                if self._cap == 0:
                    self._size_handles()
            if self.use_graph and self.pipelined and timing is None and target_ready is None:
                loss = self._step_graphed()
            else:
                loss = self._step_body(timing, target_ready)
        if sync_loss:
            val = float(loss)
            if self.pipelined and self._check_overflow(block=True):
                return self.step(sync_loss=True, timing=timing, target_ready=target_ready)
            return val
        return loss

    def step_with_targets(self, color, depth, mask, sync_loss=False):
        """One window iteration whose targets -- colour ``[n, H, W, 3]``, depth
        and valid mask ``[n, H, W]`` of this rank's views in ``views`` order,
        in pinned host memory, dtypes as ``tcolor`` / ``tdepth`` / ``tmask`` --
        are uploaded on a copy stream as part of the step: each view
        composites once its own target has arrived (no view's preparation
        waits for them).  Returns the loss like :meth:`step`.  With
        ``use_graph`` the uploads and the step are captured once for these
        host buffers and replayed."""
        n = len(self.views)
        for name, t, ref in (("color", color, self.tcolor), ("depth", depth, self.tdepth),
                             ("mask", mask, self.tmask)):
            if t.is_cuda or tuple(t.shape) != (n,) + tuple(ref.shape[1:]) or t.dtype != ref.dtype:
                raise ValueError(f"step_with_targets: {name} must be a host tensor "
                                 f"{(n,) + tuple(ref.shape[1:])} {ref.dtype}")
            if self.use_graph and not t.is_pinned():
                raise ValueError(f"step_with_targets: {name} must be in pinned memory "
                                 "(the copies are captured in a CUDA graph)")
        with torch.cuda.device(self.dev):
            if self.pipelined:
                self._check_overflow(block=False)
                if self._cap == 0:
                    self._size_handles()
            if self.use_graph and self.pipelined:
                loss = self._host_step_graphed(color, depth, mask)
            else:
                loss = self._host_step_body(color, depth, mask)
        if sync_loss:
            val = float(loss)
            if self.pipelined and self._check_overflow(block=True):
                return self.step_with_targets(color, depth, mask, sync_loss=True)
            return val
        return loss

    def _host_step_body(self, color, depth, mask, host_flag=None):
        main = torch.cuda.current_stream(self.dev)
        if self._copy is None:
            self._copy = torch.cuda.Stream(self.dev)
        start = torch.cuda.Event()
        start.record(main)  # the previous step no longer reads the targets
        self._copy.wait_event(start)
        ready = {}
        with torch.cuda.stream(self._copy):
            for j, v in enumerate(self.views):
                self.tcolor[v].copy_(color[j], non_blocking=True)
                self.tdepth[v].copy_(depth[j], non_blocking=True)
                self.tmask[v].copy_(mask[j], non_blocking=True)
                ready[v] = torch.cuda.Event()
                ready[v].record(self._copy)
        loss = self._step_body(None, ready, host_flag=host_flag)
        main.wait_stream(self._copy)
        return loss

    def _host_step_graphed(self, color, depth, mask):
        key = (color.data_ptr(), depth.data_ptr(), mask.data_ptr())
        if self._hgraph is None or self._hgraph_key != key:
            loss = self._host_step_body(color, depth, mask)  # sizes and allocations settle
            self._hgraph_host = torch.empty(1, dtype=torch.int32).pin_memory()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._hgraph_loss = self._host_step_body(color, depth, mask,
                                                         host_flag=self._hgraph_host)
            self._hgraph, self._hgraph_key = g, key
            return loss
        self._hgraph.replay()
        ev = torch.cuda.Event()
        ev.record()
        self._pending.append((ev, self._hgraph_host, self.adam_enabled))
        return self._hgraph_loss

    def _step_graphed(self):
        """Replay the captured step (the first call runs the step eagerly --
        sizes and allocations settle -- and captures it for the next calls)."""
        if self._graph is None:
            loss = self._step_body(None, None)
            self._graph_host = torch.empty(1, dtype=torch.int32).pin_memory()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._graph_loss = self._step_body(None, None, host_flag=self._graph_host)
            self._graph = g
            return loss
        self._graph.replay()
        ev = torch.cuda.Event()
        ev.record()
        self._pending.append((ev, self._graph_host, self.adam_enabled))
        return self._graph_loss

    def _step_body(self, timing=None, target_ready=None, host_flag=None):
        self.loss_acc.zero_()
        self._flag.zero_()
        adam = self.adam_enabled
        with torch.cuda.device(self.dev):
            if self.pipelined:
                self._render_pipelined(timing, target_ready)
            else:
                main = torch.cuda.current_stream(self.dev)
                if target_ready is not None:
                    for ev in target_ready.values():
                        main.wait_event(ev)
                for v in self.views:
                    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                    ev[0].record(main)
                    r = self.raster
                    ns, npairs = r.prepare(self._frames[v], self.cam, want_coef=True)
                    self._counts[v, 0], self._counts[v, 1] = ns, npairs
                    ev[1].record(main)
                    if ns:
                        split = []
                        self._composite(r, v, main,
                                        marks=lambda: (ev[2].record(main), split.append(1)))
                        ev[3].record(main)
                        if timing is not None:
                            timing.append(("prep", ev[0], ev[1], v))
                            if split:
                                timing += [("fwd", ev[1], ev[2], v), ("bwd", ev[2], ev[3], v)]
                            else:
                                timing.append(("fb", ev[1], ev[3], v))
            if self.adam_enabled and self._sharded():
                self._sharded_update()
            else:
                allreduce_window(self.grad, self.loss_acc, self.pg)
                if self.adam_enabled:  # (tests inspect the reduced gradient with it off)
                    self.apply_adam()
            if self.pipelined:
                capturing = host_flag is not None
                host = host_flag if capturing else torch.empty(1, dtype=torch.int32).pin_memory()
                host.copy_(self._flag, non_blocking=True)
                if not capturing:
                    ev = torch.cuda.Event()
                    ev.record()
                    self._pending.append((ev, host, adam))
        n_color = 3.0 * self.HW
        nd, has_d = self._nd
        ssim_term = (1.0 - self.loss_acc[:, 2] / n_color) if self.cfg.tau != 0.0 else 0.0
        return (self.cfg.rho * self.loss_acc[:, 0] / n_color + self.cfg.tau * ssim_term +
                self.cfg.sigma * torch.where(has_d, self.loss_acc[:, 1] / nd,
                                             torch.zeros_like(nd))).sum()

    def apply_adam(self):
        """One Adam step of the whole window from the (reduced) gradient
        buffer, which it consumes (zeroes)."""
        with torch.cuda.device(self.dev):
            self._t_dev.add_(1 - self._flag)  # (a step that overflowed does not count)
            _adam(self.planes, self.grad, self.m, self.v, self.F, self.HW, self.cfg, 1, False,
                  skip=self._flag, t_dev=self._t_dev)

    def _sharded(self) -> bool:
        dist = torch.distributed
        if not (self.shard_adam and dist.is_available() and dist.is_initialized()):
            return False
        world = dist.get_world_size(self.pg)
        return world > 1 and self.F % world == 0

    def _sharded_update(self):
        """Reduce-scatter -> Adam on this rank's frames -> all-gather."""
        dist = torch.distributed
        if self._shard is None:
            world, rank = dist.get_world_size(self.pg), dist.get_rank(self.pg)
            f0, f1 = frame_shard(self.F, rank, world)
            local = torch.empty(((f1 - f0) * self.HW, 8), dtype=torch.float32, device=self.dev)
            stage = torch.empty((f1 - f0,) + tuple(self.planes.shape[1:]),
                                dtype=self.planes.dtype, device=self.dev)
            self._shard = (f0, f1, local, stage)
        f0, f1, local, stage = self._shard
        reduce_scatter_window(self.grad, local, self.loss_acc, self.pg)
        self.grad.zero_()  # this step's contributions are all in the scattered blocks
        self._t_dev.add_(1 - self._flag)
        _adam(self.planes[f0:f1], local, self.m[f0:f1], self.v[f0:f1], f1 - f0, self.HW,
              self.cfg, 1, False, skip=self._flag, t_dev=self._t_dev)
        allgather_planes(self.planes, stage, f0, f1, self.pg)

    def grads_numpy(self):
        """Current gradient buffer as per-frame MapGradients-like dicts (host)."""
        g = self.grad.view(self.F, self.H, self.W, 8).double().cpu().numpy()
        return [dict(delta=g[i, ..., 0], radius=g[i, ..., 1], opacity_logit=g[i, ..., 2],
                     color=g[i, ..., 3:6]) for i in range(self.F)]


# ---------------------------------------------------------------- per-frame driver


def target_schedule(iters: int, n_neighbors: int, min_current_fraction: float,
                    seed: int = 0) -> list:
    """mapper.py:175-194: slot 0 is the current frame, 1..n its neighbours;
    strict alternation (current on even slots, neighbours round-robin from
    ``seed`` on odd slots) with extra current slots whenever the current
    frame's share would drop below ``min_current_fraction``."""
    out, n_cur, n_nb = [], 0, 0
    for i in range(iters):
        if n_neighbors == 0 or n_cur < min_current_fraction * (i + 1) or i % 2 == 0:
            out.append(0)
            n_cur += 1
        else:
            out.append(1 + (seed + n_nb) % n_neighbors)
            n_nb += 1
    return out


def assemble_base_depth(frame, pose: Pose, neighbor_maps) -> np.ndarray:
    """mapper.py:197-214: sensor depth where valid; holes covered by the
    neighbours (accumulated alpha > 0.5) take their alpha-normalised rendered
    depth (GPU splat); remaining holes are inpainted (GPU Jacobi)."""
    from .depthfill import inpaint_depth
    from .rasterizer import splat
    valid = np.asarray(frame.valid_mask, dtype=bool)
    base = np.where(valid, np.asarray(frame.depth, dtype=np.float64), 0.0)
    if valid.all():
        return base
    if neighbor_maps:
        out = splat(list(neighbor_maps), pose, frame.intrinsics, normalize_depth=True)
        a = out.alpha.cpu().numpy()
        d = out.depth.cpu().numpy()
        fill = (~valid) & (a > 0.5) & (d > 0)
        base[fill] = d[fill]
    if (base > 0).all():
        return base
    return inpaint_depth(base, base > 0)


def map_frame(frame, pose: Pose, neighbors, cfg: MapperConfig, seed: int = 0):
    """mapper.py:217-247: fit a frame's Gaussian map at a fixed pose against a
    deterministic schedule of targets (the frame and its neighbours, whose
    maps are rendered alongside but never updated).  ``neighbors`` holds
    (frame, pose, PixelGaussianMap) triples; returns (map, losses)."""
    from .gaussians import init_gaussians
    if not np.asarray(frame.valid_mask, dtype=bool).any():
        raise ValueError(f"frame {frame.index} has no valid depth to map")
    neighbors = [n for n in neighbors if np.asarray(n[0].valid_mask, dtype=bool).any()]
    neighbor_maps = [m for _, _, m in neighbors]
    base = assemble_base_depth(frame, pose, neighbor_maps)
    dev = neighbor_maps[0].planes.device if neighbor_maps else None
    gmap = init_gaussians(frame, pose, base_depth=base, device=dev)
    opt = MapOptimizer(gmap, cfg)
    losses = []
    for slot in target_schedule(cfg.mapping_iters, len(neighbors), cfg.min_current_fraction, seed):
        t_frame, t_pose = (frame, pose) if slot == 0 else neighbors[slot - 1][:2]
        losses.append(mapping_step(gmap, opt, t_frame, t_pose, neighbor_maps, cfg).total)
    return gmap, losses
