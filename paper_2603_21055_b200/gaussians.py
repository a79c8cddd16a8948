"""Pixel-aligned Gaussian maps, device-resident.

Mirrors /root/reference/pkg/src/raysplat/gaussians.py:49-115.  One Gaussian
per active pixel sits on its pixel ray at depth ``|base_depth + delta|``; the
learnable attributes are colour, log radius, opacity logit and the depth
offset.  B200 layout: one ``planes`` tensor ``[7, H, W]`` (fp64 for drop-in
maps, as the reference; fp32 in the window engine, as BASELINE) in the file
plane order of gaussians.py:9-13 (base_depth, delta, log_radius,
opacity_logit, R, G, B) plus a uint8 ``[H, W]`` active mask, both on the GPU.
The reference attribute names are views into ``planes``, so code written
against the reference (``gmap.opacity_logit[:] = 20.0``) keeps working.
"""

from __future__ import annotations

import numpy as np
import torch

from .geometry import Intrinsics, Pose

PLANES = ("base_depth", "delta", "log_radius", "opacity_logit", "r", "g", "b")


def _device(device=None):
    if device is not None:
        return torch.device(device)
    return torch.device("cuda", torch.cuda.current_device())


def _shape(x):
    return tuple(x.shape) if hasattr(x, "shape") else np.shape(x)


def _as_tensor(x, dtype, device):
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=dtype)
    return torch.as_tensor(np.asarray(x), dtype=dtype, device=device)


class PixelGaussianMap:
    """Same constructor and fields as raysplat.gaussians.PixelGaussianMap."""

    def __init__(self, frame_index, pose: Pose, intrinsics: Intrinsics, base_depth, delta, color,
                 log_radius, opacity_logit, active_mask, device=None, dtype=torch.float64):
        if dtype not in (torch.float32, torch.float64):
            raise ValueError("planes dtype must be float32 (window engine) or float64 (drop-in)")
        dev = _device(device)
        base = _as_tensor(base_depth, dtype, dev)
        if base.dim() != 2:
            raise ValueError("base_depth must be (H, W)")
        h, w = base.shape
        for name, val in (("delta", delta), ("log_radius", log_radius),
                          ("opacity_logit", opacity_logit)):
            if tuple(_shape(val)) != (h, w):
                raise ValueError(f"{name} shape differs from base_depth")
        if tuple(_shape(color)) != (h, w, 3):
            raise ValueError("color must be (H, W, 3)")
        if tuple(_shape(active_mask)) != (h, w):
            raise ValueError("active_mask shape differs from base_depth")
        planes = torch.empty((7, h, w), dtype=dtype, device=dev)
        planes[0] = base
        planes[1] = _as_tensor(delta, dtype, dev)
        planes[2] = _as_tensor(log_radius, dtype, dev)
        planes[3] = _as_tensor(opacity_logit, dtype, dev)
        planes[4:7] = _as_tensor(color, dtype, dev).permute(2, 0, 1)
        self._init(frame_index, pose, intrinsics, planes,
                   _as_tensor(active_mask, torch.bool, dev).to(torch.uint8))

    def _init(self, frame_index, pose, intrinsics, planes, mask):
        self.frame_index = int(frame_index)
        self.pose = pose
        self.intrinsics = intrinsics
        self.planes = planes.contiguous()
        self.mask_u8 = mask.contiguous()

    @classmethod
    def from_planes(cls, frame_index, pose, intrinsics, planes: torch.Tensor, mask_u8: torch.Tensor):
        """Wrap existing device storage (e.g. a slice of a window tensor) without copying."""
        obj = cls.__new__(cls)
        if planes.dtype not in (torch.float32, torch.float64) or planes.dim() != 3 \
                or planes.shape[0] != 7:
            raise ValueError("planes must be a [7, H, W] float32/float64 tensor")
        if not planes.is_contiguous():
            raise ValueError("planes must be contiguous")
        obj.frame_index = int(frame_index)
        obj.pose = pose
        obj.intrinsics = intrinsics
        obj.planes = planes
        obj.mask_u8 = mask_u8
        return obj

    # reference field names (views into planes)
    @property
    def base_depth(self):
        return self.planes[0]

    @property
    def delta(self):
        return self.planes[1]

    @property
    def log_radius(self):
        return self.planes[2]

    @property
    def opacity_logit(self):
        return self.planes[3]

    @property
    def color(self):
        return self.planes[4:7].permute(1, 2, 0)

    @property
    def active_mask(self):
        return self.mask_u8.bool()

    @property
    def shape(self):
        return tuple(self.planes.shape[1:])

    @property
    def radius(self):
        return torch.exp(self.log_radius.double())

    @property
    def opacity(self):
        return torch.sigmoid(self.opacity_logit.double())

    @property
    def adjusted_depth(self):
        return (self.base_depth.double() + self.delta.double()).abs()

    def num_active(self) -> int:
        return int(self.mask_u8.sum().item())

    def to_numpy(self):
        """Host copy with the reference's field names (fp64 arrays)."""
        from types import SimpleNamespace
        p = self.planes.double().cpu().numpy()
        return SimpleNamespace(
            frame_index=self.frame_index, pose=self.pose, intrinsics=self.intrinsics,
            base_depth=p[0].copy(), delta=p[1].copy(), log_radius=p[2].copy(),
            opacity_logit=p[3].copy(), color=np.ascontiguousarray(p[4:7].transpose(1, 2, 0)),
            active_mask=self.mask_u8.cpu().numpy().astype(bool))


def init_gaussians(frame, pose: Pose, base_depth=None, device=None,
                   dtype=torch.float64) -> PixelGaussianMap:
    """raysplat/gaussians.py:91-115: r = D/fx, opacity 0.5, zero offset, frame colour."""
    base = np.asarray(frame.depth if base_depth is None else base_depth, dtype=np.float64)
    active = base > 0
    safe = np.where(active, base, 1.0)
    return PixelGaussianMap(
        frame_index=frame.index, pose=pose, intrinsics=frame.intrinsics,
        base_depth=np.where(active, base, 0.0), delta=np.zeros_like(base),
        color=np.asarray(frame.color, dtype=np.float64), log_radius=np.log(safe / frame.intrinsics.fx),
        opacity_logit=np.zeros_like(base), active_mask=active, device=device, dtype=dtype)


# ---------------------------------------------------------------- map files
# raysplat/gaussians.py:1-15 layout, little-endian: b"RSGM", u32 version 1,
# u32 height, u32 width, i64 frame index, 12 f64 pose entries (rotation
# row-major, translation), 7 f32 planes (base_depth, delta, radius,
# opacity_logit, R, G, B), one u8 active flag per pixel.

MAP_MAGIC = b"RSGM"
MAP_VERSION = 1
_MAP_HEAD = "<4sIIIq"


class GaussianMapError(ValueError):
    """A malformed or truncated map file (gaussians.py)."""


def save_gaussian_map(path, gmap: PixelGaussianMap) -> None:
    """gaussians.py:118-136."""
    import struct
    h, w = gmap.shape
    p = gmap.planes.double().cpu().numpy()
    planes = np.stack([p[0], p[1], np.exp(p[2]), p[3], p[4], p[5], p[6]]).astype("<f4")
    pose = np.concatenate([np.asarray(gmap.pose.rotation, dtype=np.float64).reshape(9),
                           np.asarray(gmap.pose.translation, dtype=np.float64)]).astype("<f8")
    with open(path, "wb") as f:
        f.write(struct.pack(_MAP_HEAD, MAP_MAGIC, MAP_VERSION, h, w, int(gmap.frame_index)))
        f.write(pose.tobytes())
        f.write(planes.tobytes())
        f.write(gmap.mask_u8.cpu().numpy().astype(np.uint8).tobytes())


def load_gaussian_map(path, intrinsics: Intrinsics, device=None,
                      dtype=torch.float64) -> PixelGaussianMap:
    """gaussians.py:139-180: errors name the offending path."""
    import struct
    from pathlib import Path
    path = Path(path)
    blob = path.read_bytes()
    head = struct.calcsize(_MAP_HEAD)
    if len(blob) < head + 96:
        raise GaussianMapError(f"gaussian map file too short: {path}")
    magic, version, h, w, frame_index = struct.unpack_from(_MAP_HEAD, blob, 0)
    if magic != MAP_MAGIC:
        raise GaussianMapError(f"bad magic in gaussian map file: {path}")
    if version != MAP_VERSION:
        raise GaussianMapError(f"unsupported gaussian map version {version} in {path}")
    want = head + 96 + 28 * h * w + h * w
    if len(blob) != want:
        raise GaussianMapError(f"gaussian map file {path} has {len(blob)} bytes, expected {want}")
    pose = np.frombuffer(blob, dtype="<f8", count=12, offset=head)
    planes = np.frombuffer(blob, dtype="<f4", count=7 * h * w, offset=head + 96).reshape(7, h, w)
    mask = np.frombuffer(blob, dtype=np.uint8, count=h * w, offset=head + 96 + 28 * h * w)
    radius = planes[2].astype(np.float64)
    if (radius <= 0).any():
        raise GaussianMapError(f"non-positive radius in gaussian map file: {path}")
    return PixelGaussianMap(
        int(frame_index), Pose(pose[:9].reshape(3, 3).copy(), pose[9:].copy()), intrinsics,
        planes[0].astype(np.float64), planes[1].astype(np.float64),
        np.stack([planes[4], planes[5], planes[6]], axis=-1).astype(np.float64),
        np.log(radius), planes[3].astype(np.float64), mask.reshape(h, w).astype(bool),
        device=device, dtype=dtype)
