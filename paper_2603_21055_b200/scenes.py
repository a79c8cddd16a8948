"""Seeded synthetic RGBD inputs for the BASELINE.json configurations C1-C5.

The datasets the paper measures on (Replica, TUM) are not available here, so
seeded ray-cast scenes with the same image sizes, intrinsics, Gaussian
counts and parameter distributions stand in for them.
The primitives (rectangles, axis-aligned boxes, spheres, flat or checker
albedo; camera-frame z as depth) restate the ray caster of
raysplat/synthetic.py:34-199.  Casting runs in torch fp64 so the 1200x680x32
stress scene can be generated on the GPU; it is input generation, not part of
the measured hot path.

Seeds (fixed): scene geometry 0, learnable parameters 1, target parameters 2,
SE(3) query perturbation 3, depth noise rng([4, frame]).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .geometry import Intrinsics, Pose, se3_exp

_Z_NEAR = 0.01


@dataclass(frozen=True)
class Checker:
    color_a: tuple
    color_b: tuple
    cell: float = 0.2


@dataclass(frozen=True)
class Rect:
    origin: tuple
    edge_u: tuple
    edge_v: tuple
    albedo: object


@dataclass(frozen=True)
class Box:
    lo: tuple
    hi: tuple
    albedo: object


@dataclass(frozen=True)
class Sphere:
    center: tuple
    radius: float
    albedo: object


@dataclass
class Frame:
    """One RGBD observation (the fields of raysplat/datasets.py:44-60)."""

    color: np.ndarray      # (H, W, 3) float32
    depth: np.ndarray      # (H, W) float32, 0 = invalid
    valid_mask: np.ndarray  # (H, W) bool
    intrinsics: Intrinsics
    timestamp: float = 0.0
    index: int = 0


def _t(x, dev):
    return torch.as_tensor(np.asarray(x, dtype=np.float64), dtype=torch.float64, device=dev)


def _hit_rect(p, o, d):
    dev = d.device
    org, eu, ev = _t(p.origin, dev), _t(p.edge_u, dev), _t(p.edge_v, dev)
    n = torch.linalg.cross(eu, ev)
    den = d @ n
    safe = torch.where(den.abs() > 1e-12, den, torch.ones_like(den))
    s = torch.where(den.abs() > 1e-12, ((org - o) @ n) / safe, torch.full_like(den, np.inf))
    hit = o + s[:, None] * d
    q = hit - org
    a = (q @ eu) / (eu @ eu)
    b = (q @ ev) / (ev @ ev)
    inside = (a >= 0) & (a <= 1) & (b >= 0) & (b <= 1) & (s > _Z_NEAR)
    return torch.where(inside, s, torch.full_like(s, np.inf))


def _hit_box(p, o, d):
    dev = d.device
    lo, hi = _t(p.lo, dev), _t(p.hi, dev)
    par = d.abs() < 1e-12
    dsafe = torch.where(par, torch.ones_like(d), d)
    t1 = (lo - o) / dsafe
    t2 = (hi - o) / dsafe
    inside = (o >= lo) & (o <= hi)
    big = torch.full_like(t1, np.inf)
    t1 = torch.where(par, torch.where(inside, -big, big), t1)
    t2 = torch.where(par, torch.where(inside, big, -big), t2)
    t_enter = torch.minimum(t1, t2).amax(dim=1)
    t_exit = torch.maximum(t1, t2).amin(dim=1)
    s = torch.where(t_enter > _Z_NEAR, t_enter, t_exit)
    valid = (t_exit >= torch.clamp(t_enter, min=_Z_NEAR)) & (s > _Z_NEAR)
    return torch.where(valid, s, torch.full_like(s, np.inf))


def _hit_sphere(p, o, d):
    oc = o - _t(p.center, d.device)
    a = (d * d).sum(1)
    b = 2.0 * (d @ oc)
    c = oc @ oc - p.radius ** 2
    disc = b * b - 4 * a * c
    ok = disc >= 0
    sq = torch.sqrt(torch.clamp(disc, min=0))
    s1 = (-b - sq) / (2 * a)
    s2 = (-b + sq) / (2 * a)
    s = torch.where(s1 > _Z_NEAR, s1, s2)
    return torch.where(ok & (s > _Z_NEAR), s, torch.full_like(s, np.inf))


_HIT = {Rect: _hit_rect, Box: _hit_box, Sphere: _hit_sphere}


def _albedo(alb, pts):
    if isinstance(alb, Checker):
        par = torch.floor(pts / alb.cell).sum(1).to(torch.int64) & 1
        a = _t(alb.color_a, pts.device)
        b = _t(alb.color_b, pts.device)
        return torch.where(par[:, None] == 0, a, b)
    return _t(alb, pts.device).expand(len(pts), 3)


def render_frame(prims, pose: Pose, intr: Intrinsics, index: int = 0, depth_noise_rel: float = 0.0,
                 device="cpu") -> Frame:
    """Ray cast one RGBD frame (raysplat/synthetic.py:150-199 semantics)."""
    dev = torch.device(device)
    u = torch.arange(intr.width, dtype=torch.float64, device=dev)
    v = torch.arange(intr.height, dtype=torch.float64, device=dev)
    vv, uu = torch.meshgrid(v, u, indexing="ij")
    rays = torch.stack([(uu - intr.cx) / intr.fx, (vv - intr.cy) / intr.fy,
                        torch.ones_like(uu)], -1).reshape(-1, 3)
    d = rays @ _t(pose.rotation, dev).T
    o = _t(pose.translation, dev)
    best = torch.full((d.shape[0],), np.inf, dtype=torch.float64, device=dev)
    prim_id = torch.full((d.shape[0],), -1, dtype=torch.int64, device=dev)
    for k, p in enumerate(prims):
        s = _HIT[type(p)](p, o, d)
        closer = s < best
        best = torch.where(closer, s, best)
        prim_id = torch.where(closer, torch.full_like(prim_id, k), prim_id)
    hit = torch.isfinite(best)
    depth = torch.where(hit, best, torch.zeros_like(best))
    color = torch.zeros_like(d)
    pts = o + depth[:, None] * d
    for k, p in enumerate(prims):
        sel = hit & (prim_id == k)
        if bool(sel.any()):
            color[sel] = _albedo(p.albedo, pts[sel])
    depth = depth.cpu().numpy()
    hit = hit.cpu().numpy()
    if depth_noise_rel > 0.0:
        rng = np.random.default_rng([4, index])
        depth = depth * (1.0 + depth_noise_rel * rng.normal(size=depth.shape))
    hit = hit & (depth > 0)
    depth = np.where(hit, depth, 0.0)
    h, w = intr.height, intr.width
    return Frame(color=color.cpu().numpy().reshape(h, w, 3).astype(np.float32),
                 depth=depth.reshape(h, w).astype(np.float32), valid_mask=hit.reshape(h, w),
                 intrinsics=intr, timestamp=index / 30.0, index=index)


# ---------------------------------------------------------------- configs


@dataclass
class MapParams:
    """fp32-representable parameter planes of one pixel-aligned map."""

    base_depth: np.ndarray
    delta: np.ndarray
    log_radius: np.ndarray
    opacity_logit: np.ndarray
    color: np.ndarray
    active_mask: np.ndarray


def _f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def random_params(frame: Frame, seed: int) -> MapParams:
    """C1 parameter draw: r = D/fx, logit ~ N(2, 0.5), rgb ~ U[0,1], delta ~ N(0, 0.01 m)."""
    rng = np.random.default_rng(seed)
    h, w = frame.depth.shape
    base = np.asarray(frame.depth, dtype=np.float64)
    active = base > 0
    safe = np.where(active, base, 1.0)
    return MapParams(
        base_depth=_f32(np.where(active, base, 0.0)),
        delta=_f32(rng.normal(0.0, 0.01, (h, w))),
        log_radius=_f32(np.log(safe / frame.intrinsics.fx)),
        opacity_logit=_f32(rng.normal(2.0, 0.5, (h, w))),
        color=_f32(rng.uniform(0.0, 1.0, (h, w, 3))),
        active_mask=active,
    )


def init_params(frame: Frame) -> MapParams:
    """raysplat/gaussians.py:91-115: r = D/fx, opacity 0.5, zero offset, frame colour."""
    base = np.asarray(frame.depth, dtype=np.float64)
    active = base > 0
    safe = np.where(active, base, 1.0)
    return MapParams(
        base_depth=_f32(np.where(active, base, 0.0)),
        delta=np.zeros_like(base),
        log_radius=_f32(np.log(safe / frame.intrinsics.fx)),
        opacity_logit=np.zeros_like(base),
        color=_f32(frame.color),
        active_mask=active,
    )


def plane_spheres_scene(seed: int = 0):
    """Ground plane with depth spanning [1, 3] m across the view, plus 3 spheres."""
    rng = np.random.default_rng(seed)
    floor = Checker((0.55, 0.45, 0.35), (0.8, 0.72, 0.6), cell=0.25)
    # plane z = 1.5 - y: depth 3 m at the top image edge, 1 m at the bottom
    prims = [Rect((-6.0, -6.0, 7.5), (12.0, 0.0, 0.0), (0.0, 12.0, -12.0), floor)]
    for _ in range(3):
        r = float(rng.uniform(0.3, 0.6))
        c = (float(rng.uniform(-0.6, 0.6)), float(rng.uniform(-0.3, 0.3)), 0.0)
        zc = 1.5 - c[1] - r * 1.2 - float(rng.uniform(0.0, 0.3))
        prims.append(Sphere((c[0], c[1], zc), r, tuple(rng.uniform(0.2, 0.9, 3))))
    return prims


def corner_spheres_scene(seed: int = 0):
    """C2: floor, back wall and side wall (a well-posed registration target)
    plus 3 spheres of radius 0.3-0.6 m; depth spans ~1-3 m."""
    rng = np.random.default_rng(seed)
    grey = Checker((0.5, 0.5, 0.5), (0.7, 0.7, 0.7), cell=0.3)
    prims = [Rect((-3.0, 0.8, -1.0), (6.0, 0.0, 0.0), (0.0, 0.0, 6.0), grey),
             Rect((-3.0, -2.0, 3.0), (6.0, 0.0, 0.0), (0.0, 2.8, 0.0), grey),
             Rect((-1.4, -2.0, -1.0), (0.0, 2.8, 0.0), (0.0, 0.0, 4.0), grey)]
    for _ in range(3):
        r = float(rng.uniform(0.3, 0.6))
        prims.append(Sphere((float(rng.uniform(-0.6, 0.8)), float(rng.uniform(-0.3, 0.8 - r)),
                             float(rng.uniform(1.5, 2.6))), r, tuple(rng.uniform(0.2, 0.9, 3))))
    return prims


def room_scene(seed: int = 0, n_spheres: int = 20):
    """Five box walls (floor, ceiling, back, left, right) plus random spheres."""
    rng = np.random.default_rng(seed)
    wx, wy, z0, z1 = 3.0, 1.5, -1.0, 6.0
    chk = [Checker(tuple(rng.uniform(0.3, 0.6, 3)), tuple(rng.uniform(0.6, 0.9, 3)),
                   cell=float(rng.uniform(0.2, 0.4))) for _ in range(5)]
    prims = [
        Rect((-wx, wy, z0), (2 * wx, 0, 0), (0, 0, z1 - z0), chk[0]),    # floor (y down)
        Rect((-wx, -wy, z0), (2 * wx, 0, 0), (0, 0, z1 - z0), chk[1]),   # ceiling
        Rect((-wx, -wy, z1), (2 * wx, 0, 0), (0, 2 * wy, 0), chk[2]),    # back wall
        Rect((-wx, -wy, z0), (0, 2 * wy, 0), (0, 0, z1 - z0), chk[3]),   # left
        Rect((wx, -wy, z0), (0, 2 * wy, 0), (0, 0, z1 - z0), chk[4]),    # right
    ]
    for _ in range(n_spheres):
        r = float(rng.uniform(0.15, 0.5))
        c = (float(rng.uniform(-wx + r, wx - r)), float(rng.uniform(-wy + r, wy - r)),
             float(rng.uniform(1.5, z1 - r)))
        prims.append(Sphere(c, r, tuple(rng.uniform(0.1, 0.95, 3))))
    return prims


def corridor_scene(seed: int = 0, n_boxes: int = 100, length: float = 24.0):
    """A 20 m-plus corridor lined with random boxes (the C5 stress scene)."""
    rng = np.random.default_rng(seed)
    wx, wy, z0, z1 = 2.0, 1.4, -1.0, length
    walls = [Checker(tuple(rng.uniform(0.3, 0.6, 3)), tuple(rng.uniform(0.6, 0.9, 3)),
                     cell=0.3) for _ in range(5)]
    prims = [
        Rect((-wx, wy, z0), (2 * wx, 0, 0), (0, 0, z1 - z0), walls[0]),
        Rect((-wx, -wy, z0), (2 * wx, 0, 0), (0, 0, z1 - z0), walls[1]),
        Rect((-wx, -wy, z1), (2 * wx, 0, 0), (0, 2 * wy, 0), walls[2]),
        Rect((-wx, -wy, z0), (0, 2 * wy, 0), (0, 0, z1 - z0), walls[3]),
        Rect((wx, -wy, z0), (0, 2 * wy, 0), (0, 0, z1 - z0), walls[4]),
    ]
    for _ in range(n_boxes):
        size = rng.uniform(0.15, 0.6, 3)
        side = rng.choice([-1.0, 1.0])
        x = side * float(rng.uniform(0.8, wx - size[0] / 2))
        y = float(rng.uniform(-wy + size[1] / 2, wy - size[1] / 2))
        z = float(rng.uniform(1.0, z1 - 1.0))
        lo = (x - size[0] / 2, y - size[1] / 2, z - size[2] / 2)
        hi = (x + size[0] / 2, y + size[1] / 2, z + size[2] / 2)
        prims.append(Box(lo, hi, tuple(rng.uniform(0.1, 0.95, 3))))
    return prims


def trajectory(n: int, step_m: float = 0.05, step_deg: float = 2.0, yaw_sweep: bool = True):
    """Smooth trajectory with 5 cm / 2 degree steps."""
    poses = []
    for i in range(n):
        ang = np.deg2rad(step_deg) * (i if not yaw_sweep else (i - (n - 1) / 2))
        poses.append(se3_exp([0.0, ang, 0.0, step_m * i, 0.0, 0.02 * i]))
    return poses


@dataclass
class WindowConfig:
    name: str
    intr: Intrinsics
    poses: list
    frames: list
    params: list = field(default_factory=list)

    @property
    def n_gaussians(self):
        return sum(int(p.active_mask.size) for p in self.params)


C1_INTR = dict(fx=120.0, fy=120.0, cx=80.0, cy=60.0, width=160, height=120)
C2_INTR = dict(fx=240.0, fy=240.0, cx=159.5, cy=119.5, width=320, height=240)
C3_INTR = dict(fx=525.0, fy=525.0, cx=319.5, cy=239.5, width=640, height=480)
C4_INTR = dict(fx=600.0, fy=600.0, cx=599.5, cy=339.5, width=1200, height=680)


def config_c1(device="cpu"):
    """C1: 160x120 single frame, one random map (seed 1) and a target draw (seed 2)."""
    intr = Intrinsics(**C1_INTR)
    frame = render_frame(plane_spheres_scene(0), Pose.identity(), intr, 0, device=device)
    return intr, frame, random_params(frame, 1), random_params(frame, 2)


def config_render_init(device="cpu", angle_deg=1.0, shift_m=0.02, seed=6, intr_kw=None,
                       scene=None):
    """Render-based pose initialisation case (tracker.py:354-426): the map of
    frame A (identity pose, reference init_gaussians parameters) and a query
    frame B of the same scene (default: C1) under a seeded SE(3) offset."""
    intr = Intrinsics(**(intr_kw or C1_INTR))
    prims = scene if scene is not None else plane_spheres_scene(0)
    frame_a = render_frame(prims, Pose.identity(), intr, 0, device=device)
    rng = np.random.default_rng(seed)
    axis = rng.normal(size=3)
    axis /= np.linalg.norm(axis)
    shift = rng.normal(size=3)
    shift *= shift_m / np.linalg.norm(shift)
    truth = se3_exp(np.concatenate([axis * np.deg2rad(angle_deg), shift]))
    frame_b = render_frame(prims, truth, intr, 1, device=device)
    return intr, frame_a, frame_b, init_params(frame_a), truth


def config_window(name: str, n_frames: int, intr_kw: dict, device="cpu", scene=None,
                  step_m=0.05, step_deg=2.0) -> WindowConfig:
    intr = Intrinsics(**intr_kw)
    prims = scene if scene is not None else room_scene(0)
    poses = trajectory(n_frames, step_m, step_deg)
    frames = [render_frame(prims, p, intr, i, device=device) for i, p in enumerate(poses)]
    for i, f in enumerate(frames):
        f.index = i
    return WindowConfig(name, intr, poses, frames, [init_params(f) for f in frames])


def config_c3(device="cpu", n_frames=8):
    return config_window("C3", n_frames, C3_INTR, device)


def config_c4(device="cpu", n_frames=8):
    return config_window("C4", n_frames, C4_INTR, device)


def config_c5(device="cpu", n_frames=32):
    intr = Intrinsics(**C4_INTR)
    prims = corridor_scene(0)
    poses = [se3_exp([0.0, np.deg2rad(1.0) * np.sin(i / 5.0), 0.0, 0.0, 0.0, 20.0 * i / n_frames])
             for i in range(n_frames)]
    frames = [render_frame(prims, p, intr, i, device=device) for i, p in enumerate(poses)]
    return WindowConfig("C5", intr, poses, frames, [init_params(f) for f in frames])


def config_c2(device="cpu"):
    """C2: reference frame (identity) and a query under a seeded <=2 deg / <=5 cm
    perturbation; both with 1 % multiplicative depth noise."""
    intr = Intrinsics(**C2_INTR)
    prims = corner_spheres_scene(0)
    rng = np.random.default_rng(3)
    axis = rng.normal(size=3)
    axis /= np.linalg.norm(axis)
    angle = rng.uniform(0.0, np.deg2rad(2.0))
    shift = rng.normal(size=3)
    shift = shift / np.linalg.norm(shift) * rng.uniform(0.0, 0.05)
    truth = Pose(se3_exp(np.concatenate([axis * angle, np.zeros(3)])).rotation, shift)
    ref = render_frame(prims, Pose.identity(), intr, 0, depth_noise_rel=0.01, device=device)
    qry = render_frame(prims, truth, intr, 1, depth_noise_rel=0.01, device=device)
    return intr, ref, qry, truth
