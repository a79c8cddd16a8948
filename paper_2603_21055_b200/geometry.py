"""Host-side rigid-body and pinhole math (fp64 numpy).

Restates the parts of /root/reference/pkg/src/raysplat/geometry.py the hot
paths consume: ``Pose`` (geometry.py:28-69), ``so3_exp``/``se3_exp``
(:72-82, :144-169), ``so3_log``/``se3_log`` (:120-176, used for pose
differences), ``Intrinsics`` (:190-220) and ``pixel_rays`` (:223-232).
These are per-call host scalars (a pose is 12 doubles); the per-pixel work
lives in the sm_100a kernels.  ``sym_eigh3_batch`` (geometry.py:275) is
served by the device kernel, see :func:`paper_2603_21055_b200.tracker.sym_eigh3_batch`.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_SMALL_ANGLE = 1e-8
_NEAR_PI = np.pi - 1e-3


def _skew(w: np.ndarray) -> np.ndarray:
    return np.array([[0.0, -w[2], w[1]], [w[2], 0.0, -w[0]], [-w[1], w[0], 0.0]])


@dataclass(frozen=True)
class Pose:
    """Rigid transform ``x_world = rotation @ x_cam + translation`` (geometry.py:28-69)."""

    rotation: np.ndarray
    translation: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "rotation", np.asarray(self.rotation, dtype=np.float64))
        object.__setattr__(self, "translation",
                           np.asarray(self.translation, dtype=np.float64).reshape(3))
        if self.rotation.shape != (3, 3):
            raise ValueError(f"rotation must be 3x3, got {self.rotation.shape}")

    @staticmethod
    def identity() -> "Pose":
        return Pose(np.eye(3), np.zeros(3))

    def compose(self, other: "Pose") -> "Pose":
        """``self @ other`` (apply ``other`` first)."""
        return Pose(self.rotation @ other.rotation,
                    self.rotation @ other.translation + self.translation)

    def inverse(self) -> "Pose":
        rt = self.rotation.T
        return Pose(rt, -rt @ self.translation)

    def apply(self, points: np.ndarray) -> np.ndarray:
        pts = np.asarray(points, dtype=np.float64)
        if pts.ndim == 1:
            return self.rotation @ pts + self.translation
        return pts @ self.rotation.T + self.translation

    def matrix(self) -> np.ndarray:
        m = np.eye(4)
        m[:3, :3] = self.rotation
        m[:3, 3] = self.translation
        return m

    @staticmethod
    def from_matrix(m: np.ndarray) -> "Pose":
        m = np.asarray(m, dtype=np.float64)
        return Pose(m[:3, :3].copy(), m[:3, 3].copy())


def so3_exp(w) -> np.ndarray:
    w = np.asarray(w, dtype=np.float64)
    theta = np.linalg.norm(w)
    wx = _skew(w)
    if theta < _SMALL_ANGLE:
        return np.eye(3) + wx + 0.5 * (wx @ wx)
    a = np.sin(theta) / theta
    b = (1.0 - np.cos(theta)) / (theta * theta)
    return np.eye(3) + a * wx + b * (wx @ wx)


def _left_jacobian(w: np.ndarray) -> np.ndarray:
    theta = np.linalg.norm(w)
    wx = _skew(w)
    if theta < _SMALL_ANGLE:
        return np.eye(3) + 0.5 * wx + (wx @ wx) / 6.0
    t2 = theta * theta
    b = (1.0 - np.cos(theta)) / t2
    c = (theta - np.sin(theta)) / (t2 * theta)
    return np.eye(3) + b * wx + c * (wx @ wx)


def _left_jacobian_inv(w: np.ndarray) -> np.ndarray:
    theta = np.linalg.norm(w)
    wx = _skew(w)
    if theta < _SMALL_ANGLE:
        return np.eye(3) - 0.5 * wx + (wx @ wx) / 12.0
    half = 0.5 * theta
    cot = half / np.tan(half)
    return np.eye(3) - 0.5 * wx + (1.0 - cot) / (theta * theta) * (wx @ wx)


def se3_exp(twist) -> Pose:
    """Twist ``[w; v]`` to Pose (geometry.py:165-169)."""
    twist = np.asarray(twist, dtype=np.float64).reshape(6)
    w, v = twist[:3], twist[3:]
    return Pose(so3_exp(w), _left_jacobian(w) @ v)


def _rotation_to_quaternion(r: np.ndarray) -> np.ndarray:
    t = np.trace(r)
    if t > 0.0:
        s = np.sqrt(t + 1.0) * 2.0
        q = np.array([(r[2, 1] - r[1, 2]) / s, (r[0, 2] - r[2, 0]) / s,
                      (r[1, 0] - r[0, 1]) / s, 0.25 * s])
    else:
        i = int(np.argmax(np.diag(r)))
        j, k = (i + 1) % 3, (i + 2) % 3
        s = np.sqrt(max(r[i, i] - r[j, j] - r[k, k] + 1.0, 0.0)) * 2.0
        q = np.zeros(4)
        q[i] = 0.25 * s
        q[j] = (r[j, i] + r[i, j]) / s
        q[k] = (r[k, i] + r[i, k]) / s
        q[3] = (r[k, j] - r[j, k]) / s
    q /= np.linalg.norm(q)
    return -q if q[3] < 0.0 else q


def so3_log(r) -> np.ndarray:
    r = np.asarray(r, dtype=np.float64)
    cos_theta = np.clip((np.trace(r) - 1.0) * 0.5, -1.0, 1.0)
    theta = np.arccos(cos_theta)
    if theta < _SMALL_ANGLE:
        return 0.5 * np.array([r[2, 1] - r[1, 2], r[0, 2] - r[2, 0], r[1, 0] - r[0, 1]])
    if theta >= _NEAR_PI:
        q = _rotation_to_quaternion(r)
        vn = np.linalg.norm(q[:3])
        if vn < 1e-12:
            return np.zeros(3)
        return q[:3] / vn * (2.0 * np.arctan2(vn, q[3]))
    return theta / (2.0 * np.sin(theta)) * np.array(
        [r[2, 1] - r[1, 2], r[0, 2] - r[2, 0], r[1, 0] - r[0, 1]])


def se3_log(pose: Pose) -> np.ndarray:
    w = so3_log(pose.rotation)
    return np.concatenate([w, _left_jacobian_inv(w) @ pose.translation])


def pose_difference(a: Pose, b: Pose) -> tuple[float, float]:
    """(rotation angle rad, translation distance m) between two poses."""
    rel = a.inverse().compose(b)
    return float(np.linalg.norm(so3_log(rel.rotation))), float(np.linalg.norm(rel.translation))


@dataclass(frozen=True)
class Intrinsics:
    """Pinhole camera; pixel centres at integer coordinates (geometry.py:190-220)."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    depth_scale: float = 1.0

    def __post_init__(self):
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError("focal lengths must be positive")
        if not (0 <= self.cx < self.width and 0 <= self.cy < self.height):
            raise ValueError("principal point must lie inside the image")
        if self.depth_scale <= 0:
            raise ValueError("depth_scale must be positive")


def pixel_rays(intr: Intrinsics) -> np.ndarray:
    u = np.arange(intr.width, dtype=np.float64)
    v = np.arange(intr.height, dtype=np.float64)
    uu, vv = np.meshgrid(u, v)
    rays = np.empty((intr.height, intr.width, 3))
    rays[..., 0] = (uu - intr.cx) / intr.fx
    rays[..., 1] = (vv - intr.cy) / intr.fy
    rays[..., 2] = 1.0
    return rays


def relative_pose(target: Pose, source: Pose) -> Pose:
    """``target.inverse().compose(source)`` -- the exact expression of
    rasterizer.py:94, so the fp64 bits match the reference's."""
    return target.inverse().compose(source)
