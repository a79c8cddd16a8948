"""Geometry tracking -- drop-in for /root/reference/pkg/src/raysplat/tracker.py.

Per frame, the depth image becomes oriented geometry Gaussians (K7:
window fit + closed-form 3x3 eigendecomposition), which are registered to
the world-frame set with GICP.  Each Gauss-Newton iteration is ONE fused
kernel (K8: exact 1-NN on a uniform grid, point-to-surface gate, combined
covariance, 3x3 inverse, SE(3) Jacobian and the 6x6 J^T W J / J^T W d
reduction) followed by the 6x6 solve on the host, as north_star specifies;
the step-halving costs of the reference's line search are evaluated for all
five halvings in one launch (K9) so an iteration costs two round trips.

Delta D2 (north_star): local Gaussians fit the valid pixels of a
``window x window`` neighbourhood (self excluded, at least
``min_neighbors``) instead of the K_c Euclidean nearest neighbours; the
covariance, eigenvalue floor, scale normalisation and normal orientation
are the reference's (tracker.py:158-169).  The correspondence rule (exact
Euclidean 1-NN + gate, delta D3) is the reference's.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .geometry import Pose, se3_exp

SCALE_MODES = ("ellipse", "plane", "none")
METRIC_MODES = ("point2surf", "point2point")
INIT_MODES = ("constant_speed", "render_init")
EIGVAL_FLOOR_REL = 1e-6
PLANE_SCALES = (1.0, 1.0, 1e-3)
MIN_INLIERS = 10
MAX_STEP_HALVINGS = 5


class TrackerError(ValueError):
    pass


@dataclass
class TrackerConfig:
    """tracker.py:36-60 plus the window-fit parameters of delta D2."""

    downsample_ratio: int = 10
    neighbor_count: int = 10
    max_gicp_iters: int = 30
    correspondence_dist_max: float = 0.2
    convergence_eps: float = 1e-5
    scale_mode: str = "ellipse"
    metric_mode: str = "point2surf"
    init_mode: str = "constant_speed"
    voxel_size: float = 0.02
    render_init_iters: int = 10
    render_coverage_min: float = 0.3
    window: int = 5
    min_neighbors: int = 4

    def __post_init__(self):
        if self.downsample_ratio < 1:
            raise TrackerError("downsample_ratio must be >= 1")
        if self.neighbor_count < 4:
            raise TrackerError("neighbor_count must be >= 4")
        if self.scale_mode not in SCALE_MODES:
            raise TrackerError(f"scale_mode must be one of {SCALE_MODES}")
        if self.metric_mode not in METRIC_MODES:
            raise TrackerError(f"metric_mode must be one of {METRIC_MODES}")
        if self.init_mode not in INIT_MODES:
            raise TrackerError(f"init_mode must be one of {INIT_MODES}")
        if self.window < 3 or self.window % 2 == 0:
            raise TrackerError("window must be odd and >= 3")


def _dev():
    N.load()
    return torch.device("cuda", torch.cuda.current_device())


def _t(x, dtype=torch.float64, device=None):
    dev = device or _dev()
    if isinstance(x, torch.Tensor):
        return x.to(dev, dtype).contiguous()
    return torch.as_tensor(np.asarray(x), dtype=dtype, device=dev).contiguous()


def cov_full(cov6: torch.Tensor) -> torch.Tensor:
    c = cov6
    return torch.stack([c[:, 0], c[:, 1], c[:, 2], c[:, 1], c[:, 3], c[:, 4],
                        c[:, 2], c[:, 4], c[:, 5]], 1).view(-1, 3, 3)


def cov_packed(cov: torch.Tensor) -> torch.Tensor:
    return torch.stack([cov[:, 0, 0], cov[:, 0, 1], cov[:, 0, 2], cov[:, 1, 1], cov[:, 1, 2],
                        cov[:, 2, 2]], 1).contiguous()


def _cov_from(rot, scales):
    return torch.einsum("nij,nj,nkj->nik", rot, scales**2, rot)


class LocalGeomSet:
    """Oriented geometry Gaussians in one frame's camera (tracker.py:63-78), on device."""

    def __init__(self, centers, rotations, scales, normals, source_frame=-1, cov6=None,
                 pixel=None):
        self.centers = _t(centers)
        self.rotations = _t(rotations)
        self.scales = _t(scales)
        self.normals = _t(normals)
        self.source_frame = source_frame
        self.pixel = pixel
        self.cov6 = cov6 if cov6 is not None else cov_packed(_cov_from(self.rotations,
                                                                        self.scales))

    def __len__(self) -> int:
        return int(self.centers.shape[0])

    def covariances(self) -> torch.Tensor:
        return cov_full(self.cov6)


def sym_eigh3_batch(mats):
    """geometry.py:275-353 on device: (rotations (N,3,3), eigenvalues (N,3) descending)."""
    m = _t(mats).reshape(-1, 9)
    n = m.shape[0]
    rot = torch.empty((n, 9), dtype=torch.float64, device=m.device)
    vals = torch.empty((n, 3), dtype=torch.float64, device=m.device)
    N.call("sgad_sym_eigh3", m.data_ptr(), n, rot.data_ptr(), vals.data_ptr(), N.stream_ptr())
    return rot.view(n, 3, 3), vals


def fit_local(depth, mask, intr, stride=1, window=5, min_neighbors=4, scale_mode="ellipse",
              source_frame=-1) -> LocalGeomSet:
    """K7 on a device depth image (delta D2 window fit)."""
    dev = _dev()
    d = _t(depth, torch.float32, dev)
    mk = _t(mask, torch.uint8, dev)
    h, w = d.shape
    cap = ((h + stride - 1) // stride) * ((w + stride - 1) // stride)
    c = torch.empty((cap, 3), dtype=torch.float64, device=dev)
    cov = torch.empty((cap, 6), dtype=torch.float64, device=dev)
    nrm = torch.empty((cap, 3), dtype=torch.float64, device=dev)
    rot = torch.empty((cap, 9), dtype=torch.float64, device=dev)
    sc = torch.empty((cap, 3), dtype=torch.float64, device=dev)
    pix = torch.empty(cap, dtype=torch.int64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    N.call("sgad_track_fit", d.data_ptr(), mk.data_ptr(), h, w, float(intr.fx), float(intr.fy),
           float(intr.cx), float(intr.cy), int(stride), int(window), int(min_neighbors),
           SCALE_MODES.index(scale_mode), c.data_ptr(), cov.data_ptr(), nrm.data_ptr(),
           rot.data_ptr(), sc.data_ptr(), pix.data_ptr(), cnt.data_ptr(), N.stream_ptr())
    m = int(cnt.item())
    out = LocalGeomSet.__new__(LocalGeomSet)
    out.centers, out.cov6, out.normals = c[:m], cov[:m], nrm[:m]
    out.rotations, out.scales, out.pixel = rot[:m].view(m, 3, 3), sc[:m], pix[:m]
    out.source_frame = source_frame
    return out


def build_local_set(frame, cfg: TrackerConfig) -> LocalGeomSet:
    """tracker.py:193-230 with the window neighbourhood (delta D2)."""
    valid = np.asarray(frame.valid_mask, dtype=bool) if not isinstance(frame.valid_mask,
                                                                         torch.Tensor) \
        else frame.valid_mask.bool()
    n_valid = int(valid.sum())
    if n_valid < cfg.min_neighbors + 1:
        raise TrackerError(f"frame {frame.index}: {n_valid} valid pixels, need at least "
                           f"{cfg.min_neighbors + 1}")
    local = fit_local(frame.depth, valid, frame.intrinsics, cfg.downsample_ratio, cfg.window,
                      cfg.min_neighbors, cfg.scale_mode, frame.index)
    if len(local) == 0:
        raise TrackerError(f"frame {frame.index}: no valid pixels on the sample grid")
    return local


class GlobalGeomSet:
    """World-frame geometry Gaussians with an exact 1-NN index (tracker.py:81-133).

    Insertion keeps the reference's voxel gating (one member per cell, first
    come first served in row order) with a device hash table of occupied
    cells (csrc/voxels.cu); the members live on the device with a multi-level
    grid index rebuilt per insert, like the reference's cKDTree."""

    def __init__(self, voxel_size: float = 0.02):
        if voxel_size <= 0:
            raise TrackerError("voxel_size must be positive")
        self.voxel_size = voxel_size
        dev = _dev()
        self.centers = torch.empty((0, 3), dtype=torch.float64, device=dev)
        self.rotations = torch.empty((0, 3, 3), dtype=torch.float64, device=dev)
        self.scales = torch.empty((0, 3), dtype=torch.float64, device=dev)
        self.normals = torch.empty((0, 3), dtype=torch.float64, device=dev)
        self.cov6 = torch.empty((0, 6), dtype=torch.float64, device=dev)
        h = ctypes.c_void_p()
        N.check(N.load().sgad_geomset_create(ctypes.byref(h)))
        self._h = h
        v = ctypes.c_void_p()
        N.check(N.load().sgad_voxels_create(ctypes.byref(v)))
        self._vox = v

    def __del__(self):
        try:
            lib = N.load(require_cuda=False)
            if self._h:
                lib.sgad_geomset_destroy(self._h)
                self._h = None
            if getattr(self, "_vox", None):
                lib.sgad_voxels_destroy(self._vox)
                self._vox = None
        except Exception:
            pass

    def __len__(self) -> int:
        return int(self.centers.shape[0])

    def _gate(self, c: torch.Tensor) -> torch.Tensor:
        keep = torch.empty(c.shape[0], dtype=torch.uint8, device=c.device)
        n_keep = ctypes.c_int64()
        rc = N.load().sgad_voxels_gate(self._vox, N.ptr(c), int(c.shape[0]),
                                       float(self.voxel_size), N.ptr(keep),
                                       ctypes.byref(n_keep), N.stream_ptr())
        if rc != N.SGAD_OK:
            raise TrackerError(N.load().sgad_last_error().decode())
        return keep.bool()

    def insert(self, centers, rotations, scales, normals, cov6=None) -> int:
        """tracker.py:105-122: rows whose voxel cell is free join the set (in
        row order); returns the number added.  ``cov6`` (optional): the rows'
        packed covariances, if already computed."""
        c = _t(centers).reshape(-1, 3).contiguous()
        keep = self._gate(c)
        n = int(keep.sum())
        if n:
            rot, sc = _t(rotations)[keep], _t(scales)[keep]
            self.centers = torch.cat([self.centers, c[keep]])
            self.rotations = torch.cat([self.rotations, rot])
            self.scales = torch.cat([self.scales, sc])
            self.normals = torch.cat([self.normals, _t(normals)[keep]])
            cv = _t(cov6)[keep] if cov6 is not None else cov_packed(_cov_from(rot, sc))
            self.cov6 = torch.cat([self.cov6, cv])
            N.call("sgad_geomset_set", self._h, self.centers.data_ptr(), self.cov6.data_ptr(),
                   self.normals.data_ptr(), len(self), N.stream_ptr())
        return n

    def set_members(self, centers, cov6, normals, rotations=None, scales=None):
        """Replace the members wholesale (no voxel gating): the C2/C5 target set."""
        self.centers, self.cov6, self.normals = _t(centers), _t(cov6), _t(normals)
        self.rotations = _t(rotations) if rotations is not None else self.rotations[:0]
        self.scales = _t(scales) if scales is not None else self.scales[:0]
        # the occupancy restarts from exactly these members' cells
        lib = N.load()
        lib.sgad_voxels_destroy(self._vox)
        v = ctypes.c_void_p()
        N.check(lib.sgad_voxels_create(ctypes.byref(v)))
        self._vox = v
        if len(self):
            self._gate(self.centers.contiguous())
        N.call("sgad_geomset_set", self._h, self.centers.data_ptr(), self.cov6.data_ptr(),
               self.normals.data_ptr(), len(self), N.stream_ptr())

    def query_nearest(self, points):
        if len(self) == 0:
            raise TrackerError("global set is empty")
        q = _t(points).reshape(-1, 3)
        idx = torch.empty(q.shape[0], dtype=torch.int64, device=q.device)
        dist = torch.empty(q.shape[0], dtype=torch.float64, device=q.device)
        N.call("sgad_geomset_nearest", self._h, q.data_ptr(), q.shape[0], idx.data_ptr(),
               dist.data_ptr(), N.stream_ptr())
        return dist, idx

    def covariances(self, idx):
        return cov_full(self.cov6[idx])


def update_global_set(global_set: GlobalGeomSet, local: LocalGeomSet, pose: Pose) -> int:
    """tracker.py:233-238: the local set in the world frame (one kernel:
    centres, rotations, normals and the members' covariances in the
    reference's operation order), then the voxel-gated insertion."""
    m = len(local)
    dev = local.centers.device
    out = [torch.empty((m, 3), dtype=torch.float64, device=dev),
           torch.empty((m, 3, 3), dtype=torch.float64, device=dev),
           torch.empty((m, 3), dtype=torch.float64, device=dev),
           torch.empty((m, 6), dtype=torch.float64, device=dev)]
    rot = (ctypes.c_double * 9)(*np.asarray(pose.rotation, dtype=np.float64).reshape(9))
    tr = (ctypes.c_double * 3)(*np.asarray(pose.translation, dtype=np.float64).reshape(3))
    src = [local.centers.contiguous(), local.rotations.contiguous(), local.scales.contiguous(),
           local.normals.contiguous()]
    N.call("sgad_track_to_world", *[x.data_ptr() for x in src], m, rot, tr,
           *[x.data_ptr() for x in out], N.stream_ptr())
    centers, rotations, normals, cov6 = out
    return global_set.insert(centers, rotations, local.scales.clone(), normals, cov6=cov6)


@dataclass
class GicpDiagnostics:
    """tracker.py:241-250."""

    iterations: int = 0
    final_cost: float = float("nan")
    inlier_count: int = 0
    converged: bool = False
    failed: bool = False
    cost_pairs: list = field(default_factory=list)
    accepted_first: np.ndarray | None = None


def _sym6(h21):
    h = np.empty((6, 6))
    k = 0
    for r in range(6):
        for c in range(r, 6):
            h[r, c] = h[c, r] = h21[k]
            k += 1
    return h


class GicpSolver:
    """Device buffers + launches for one (local, global) registration."""

    def __init__(self, local: LocalGeomSet, global_set: GlobalGeomSet, cfg: TrackerConfig):
        self.local, self.g, self.cfg = local, global_set, cfg
        self.m = len(local)
        self.out = torch.empty(29, dtype=torch.float64, device=local.centers.device)
        self.costs = torch.empty(8, dtype=torch.float64, device=local.centers.device)
        self.host = torch.empty(29 + 8, dtype=torch.float64).pin_memory()
        self.metric = METRIC_MODES.index(cfg.metric_mode)
        self._warm = 0

    def linearize(self, pose: Pose):
        """K8 at ``pose``: returns (H 6x6, g 6, cost, inliers)."""
        # (later linearisations seed the exact NN search with these neighbours)
        self._eqs_launch(pose)
        h = self.host[:29]
        h.copy_(self.out)  # synchronising copy into pinned memory
        v = h.numpy()
        return _sym6(v[:21]), v[21:27].copy(), float(v[27]), int(round(v[28]))

    def _eqs_launch(self, pose: Pose):
        rot = (ctypes.c_double * 9)(*np.asarray(pose.rotation, dtype=np.float64).reshape(9))
        tr = (ctypes.c_double * 3)(*np.asarray(pose.translation, dtype=np.float64).reshape(3))
        N.call("sgad_track_normal_eqs", self.g._h, self.local.centers.data_ptr(),
               self.local.cov6.data_ptr(), self.m, rot, tr, self.metric,
               float(self.cfg.correspondence_dist_max), self._warm, self.out.data_ptr(),
               N.stream_ptr())
        self._warm = 1

    def _cost_launch(self, poses):
        arr = np.concatenate([np.concatenate([np.asarray(p.rotation).reshape(9),
                                              np.asarray(p.translation).reshape(3)])
                              for p in poses])
        buf = (ctypes.c_double * len(arr))(*arr)
        N.call("sgad_track_cost", self.g._h, self.local.centers.data_ptr(), self.m, buf,
               len(poses), self.costs.data_ptr(), N.stream_ptr())

    def costs_and_linearize(self, poses, next_pose: Pose):
        """The frozen-weight costs of the candidate poses, then (speculatively)
        the linearisation at ``next_pose``, read back with one synchronisation:
        a GN iteration whose full step is accepted needs one host round trip."""
        self._cost_launch(poses)
        if next_pose is not None:
            self._eqs_launch(next_pose)
        n = len(poses)
        self.host[29:29 + n].copy_(self.costs[:n], non_blocking=True)
        if next_pose is not None:
            self.host[:29].copy_(self.out, non_blocking=True)
        torch.cuda.current_stream(self.local.centers.device).synchronize()
        v = self.host.numpy()
        if next_pose is None:
            return v[29:29 + n].copy(), None
        return (v[29:29 + n].copy(),
                (_sym6(v[:21]), v[21:27].copy(), float(v[27]), int(round(v[28]))))

    def costs_at(self, poses):
        arr = np.concatenate([np.concatenate([np.asarray(p.rotation).reshape(9),
                                              np.asarray(p.translation).reshape(3)])
                              for p in poses])
        buf = (ctypes.c_double * len(arr))(*arr)
        N.call("sgad_track_cost", self.g._h, self.local.centers.data_ptr(), self.m, buf,
               len(poses), self.costs.data_ptr(), N.stream_ptr())
        h = self.host[29:29 + len(poses)]
        h.copy_(self.costs[:len(poses)])
        return h.numpy().copy()

    def run_device_loop(self, init: Pose):
        """The whole Gauss-Newton loop on the device (sgad_track_gicp) from
        ``init``: (result[19], systems [iters, 29], cost pairs [iters, 2],
        first acceptance flags [m] bool)."""
        it = int(self.cfg.max_gicp_iters)
        p = (ctypes.c_double * 12)(*np.concatenate([np.asarray(init.rotation, np.float64).reshape(9),
                                                    np.asarray(init.translation, np.float64).reshape(3)]))
        res = np.empty(19)
        sys_rows = np.empty((it, 29))
        pairs = np.empty((it, 2))
        acc = torch.empty(self.m, dtype=torch.uint8, device=self.local.centers.device)
        N.call("sgad_track_gicp", self.g._h, self.local.centers.data_ptr(), self.local.cov6.data_ptr(),
               self.m, p, self.metric, float(self.cfg.correspondence_dist_max), it,
               float(self.cfg.convergence_eps), self._warm, MIN_INLIERS, res.ctypes.data,
               sys_rows.ctypes.data, pairs.ctypes.data, acc.data_ptr(), N.stream_ptr())
        self._warm = 1
        return res, sys_rows, pairs, acc.bool().cpu().numpy()

    def correspondences(self):
        """The last linearisation's exact nearest neighbours (tracker.py:288 j)."""
        idx = torch.empty(self.m, dtype=torch.int64, device=self.local.centers.device)
        N.call("sgad_track_correspondences", self.g._h, idx.data_ptr(), self.m, N.stream_ptr())
        return idx.cpu().numpy()

    def accepted(self):
        acc = torch.empty(self.m, dtype=torch.uint8, device=self.local.centers.device)
        N.call("sgad_track_accepted", self.g._h, acc.data_ptr(), self.m, N.stream_ptr())
        return acc.bool().cpu().numpy()


# gicp_align runs its Gauss-Newton loop on the device (sgad_track_gicp: one
# host round trip per registration); False selects the host loop (one round
# trip per iteration), which also finishes a device loop stopped by an
# exactly singular system (numpy's lstsq fallback).
GICP_DEVICE_LOOP = True


def gicp_align(local: LocalGeomSet, global_set: GlobalGeomSet, init: Pose, cfg: TrackerConfig,
               return_systems: bool = False):
    """tracker.py:265-346: Gauss-Newton on the combined-covariance cost with
    frozen weights, at most 5 step halvings, failure below 10 inliers."""
    if len(global_set) == 0:
        raise TrackerError("global set is empty")
    diag = GicpDiagnostics()
    systems = []
    if cfg.max_gicp_iters <= 0:
        return (init, diag, systems) if return_systems else (init, diag)
    solver = GicpSolver(local, global_set, cfg)
    if not GICP_DEVICE_LOOP:
        pose = _gicp_host_loop(solver, init, init, cfg, diag, systems, 0)
        return (pose, diag, systems) if return_systems else (pose, diag)
    res, sys_rows, pairs, acc = solver.run_device_loop(init)
    diag.accepted_first = acc
    diag.iterations = int(res[13])
    diag.inlier_count = int(res[14])
    diag.converged = bool(res[15])
    diag.failed = bool(res[16])
    diag.final_cost = float(res[12])
    diag.cost_pairs = [(float(a), float(b)) for a, b in pairs[:diag.iterations]]
    systems = [(_sym6(r[:21]), r[21:27].copy(), float(r[27]), int(round(r[28])))
               for r in sys_rows[:int(res[18])]]
    pose = Pose(res[:9].reshape(3, 3).copy(), res[9:12].copy())
    singular = int(res[17])
    if singular >= 0:
        # numpy's lstsq fallback for an exactly singular system: the host
        # continues from the pose reached, re-linearising it
        systems = systems[:singular]
        pose = _gicp_host_loop(solver, pose, init, cfg, diag, systems, singular)
    return (pose, diag, systems) if return_systems else (pose, diag)


def _gicp_host_loop(solver, pose, init, cfg, diag, systems, it0):
    """The Gauss-Newton loop with the solve on the host from iteration it0 at
    ``pose`` (one host round trip per iteration: the candidate costs and,
    speculatively, the next linearisation at the full step)."""
    nxt = solver.linearize(pose)
    for it in range(it0, cfg.max_gicp_iters):
        h, g, cost_before, n_acc = nxt
        diag.inlier_count = n_acc
        if it == 0:
            diag.accepted_first = solver.accepted()
        if n_acc < MIN_INLIERS:
            diag.failed = True
            return init
        systems.append((h, g, cost_before, n_acc))
        try:
            xi = np.linalg.solve(h, -g)
        except np.linalg.LinAlgError:
            xi = np.linalg.lstsq(h, -g, rcond=None)[0]
        xis, cands = [], []
        for _ in range(MAX_STEP_HALVINGS + 1):
            xis.append(xi)
            cands.append(se3_exp(xi).compose(pose))
            xi = 0.5 * xi
        last = it + 1 == cfg.max_gicp_iters
        costs, spec = solver.costs_and_linearize(cands, None if last else cands[0])
        k = 0
        while costs[k] > cost_before and k < MAX_STEP_HALVINGS:
            k += 1
        xi, candidate, cost_after = xis[k], cands[k], float(costs[k])
        if cost_after > cost_before:
            diag.final_cost = cost_before
            break
        pose = candidate
        diag.iterations += 1
        diag.final_cost = cost_after
        diag.cost_pairs.append((cost_before, cost_after))
        if np.linalg.norm(xi) < cfg.convergence_eps:
            diag.converged = True
            break
        if not last:
            nxt = spec if k == 0 else solver.linearize(pose)
    return pose


def init_pose_constant_speed(prev: Pose, prev_prev: Pose) -> Pose:
    """tracker.py:349-351."""
    return prev.compose(prev_prev.inverse().compose(prev))


_RENDER_POOL = {}


class _RenderResiduals:
    """Residual vector of tracker.py:379-383 on the GPU: the previous frame's
    map rendered at a candidate pose (K1-K4 with preallocated images), L1
    photometric and valid-masked, weighted depth residuals concatenated into
    one device fp64 vector.  Two raster handles on two streams let a batch of
    renders (the Jacobian's 12) overlap one render's preparation with the
    previous one's compositing."""

    def __init__(self, frame, prev_map, depth_weight: float):
        from .rasterizer import Raster, camera_of
        self.intr = frame.intrinsics
        self.map = prev_map
        dev = prev_map.planes.device
        self.dev = dev
        h, w = int(self.intr.height), int(self.intr.width)
        self.tc = torch.as_tensor(np.asarray(frame.color, dtype=np.float64), device=dev)
        self.td = torch.as_tensor(np.asarray(frame.depth, dtype=np.float64), device=dev)
        self.wm = depth_weight * torch.as_tensor(np.asarray(frame.valid_mask, dtype=np.float64),
                                                 device=dev)
        self.img = [tuple(torch.empty(shape, dtype=torch.float64, device=dev)
                          for shape in ((h, w, 3), (h, w), (h, w))) for _ in range(2)]
        # raster handles and streams are reused across calls (their grow-only
        # scratch would otherwise be reallocated -- cudaFree synchronises)
        key = (dev.index, "render_init")
        if key not in _RENDER_POOL:
            _RENDER_POOL[key] = ([Raster(dev), Raster(dev)],
                                 [torch.cuda.Stream(dev), torch.cuda.Stream(dev)])
        self.rasters, self.streams = _RENDER_POOL[key]
        self.cam = camera_of(self.intr)
        self.n = 4 * h * w

    def _render(self, k: int, pose: Pose, stream) -> None:
        from .rasterizer import build_frames
        color, depth, alpha = self.img[k]
        frames = build_frames([self.map], pose, set())[0]
        r = self.rasters[k]
        ns, _ = r.prepare(frames, self.cam, stream=stream)
        if ns:
            r.forward(color, depth, alpha, stream=stream)
        else:
            with torch.cuda.stream(stream):
                color.zero_()
                depth.zero_()
                alpha.zero_()

    def _residual(self, k: int, out: torch.Tensor) -> None:
        color, depth, _ = self.img[k]
        nc = color.numel()
        torch.sub(color.reshape(-1), self.tc.reshape(-1), out=out[:nc])
        torch.mul(self.wm.reshape(-1), depth.reshape(-1) - self.td.reshape(-1), out=out[nc:])

    def batch(self, poses, out: torch.Tensor) -> torch.Tensor:
        """Residual rows out[i] for poses[i], renders alternating over the two
        handles/streams; the current stream waits for all of them."""
        main = torch.cuda.current_stream(self.dev)
        start = torch.cuda.Event()
        start.record(main)
        for st in self.streams:
            st.wait_event(start)
        for i, pose in enumerate(poses):
            k = i & 1
            st = self.streams[k]
            self._render(k, pose, st)
            with torch.cuda.stream(st):
                self._residual(k, out[i])
        for st in self.streams:
            main.wait_stream(st)
        return out

    def __call__(self, pose: Pose, out=None) -> torch.Tensor:
        r = out if out is not None else torch.empty(self.n, dtype=torch.float64, device=self.dev)
        return self.batch([pose], r[None])[0]

    def coverage(self, pose: Pose) -> float:
        self.batch([pose], torch.empty((1, self.n), dtype=torch.float64, device=self.dev))
        return float((self.img[0][2] > 0.5).double().mean())


def init_pose_render(frame, prev_map, init: Pose, iters: int = 10, depth_weight: float = 4.0,
                     coverage_min: float = 0.3):
    """tracker.py:354-426: refine ``init`` by rendering ``prev_map`` (a device
    PixelGaussianMap) against ``frame`` -- IRLS Gauss-Newton on the L1
    photometric + weighted L1 depth residuals with a central-difference
    Jacobian through the renderer.  Every render (13 per iteration plus the
    step-halving candidates) runs on the sm_100a rasterizer; residuals, the
    Jacobian and the 6x6 IRLS systems stay on the device and only the 6x6
    least-squares solves run on the host, as in the reference.  Returns
    ``(pose, ok)``; ``ok`` is False (and ``init`` returned) when the map
    covers less than ``coverage_min`` of the frame."""
    res = _RenderResiduals(frame, prev_map, depth_weight)
    if res.coverage(init) < coverage_min:
        return init, False
    pose = init
    h = 1e-4
    r = res(pose).clone()
    rows = torch.empty((12, res.n), dtype=torch.float64, device=res.dev)
    partial = torch.empty(592 * 27, dtype=torch.float64, device=res.dev)
    sums = torch.empty(27, dtype=torch.float64, device=res.dev)
    for _ in range(iters):
        # the 12 central-difference renders as one batch (residual rows)
        probes = []
        for k in range(6):
            e = np.zeros(6)
            e[k] = h
            probes += [se3_exp(e).compose(pose), se3_exp(-e).compose(pose)]
        res.batch(probes, rows)
        # IRLS on the same linearisation: weights from the predicted residuals;
        # J^T W J and J^T W r in one pass over the rows (sgad_irls_normal_eqs)
        xi = np.zeros(6)
        for _inner in range(3):
            xi_c = (ctypes.c_double * 6)(*xi)
            N.call("sgad_irls_normal_eqs", rows.data_ptr(), r.data_ptr(), int(res.n), xi_c,
                   float(h), partial.data_ptr(), sums.data_ptr(), N.stream_ptr())
            v = sums.cpu().numpy()
            xi = np.linalg.lstsq(_sym6(v[:21]), -v[21:], rcond=None)[0]
        cost = float(r.abs().sum())
        candidate = se3_exp(xi).compose(pose)
        r_cand = res(candidate)
        halvings = 0
        while float(r_cand.abs().sum()) > cost and halvings < MAX_STEP_HALVINGS:
            xi = 0.5 * xi
            candidate = se3_exp(xi).compose(pose)
            r_cand = res(candidate)
            halvings += 1
        if float(r_cand.abs().sum()) > cost:
            break
        pose, r = candidate, r_cand.clone()
        if np.linalg.norm(xi) < 1e-7:
            break
    return pose, True
