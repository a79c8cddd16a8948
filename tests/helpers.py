"""Shared test helpers: golden-array unpacking and tolerance checks."""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np

from paper_2603_21055_b200.geometry import Intrinsics, Pose

PARAM_KEYS = ("base_depth", "delta", "log_radius", "opacity_logit", "color", "active_mask")


def intr_from(arr) -> Intrinsics:
    fx, fy, cx, cy, w, h = (float(x) for x in arr)
    return Intrinsics(fx, fy, cx, cy, int(w), int(h))


def pose_from(arr) -> Pose:
    arr = np.asarray(arr, dtype=np.float64)
    return Pose(arr[:9].reshape(3, 3), arr[9:12])


def np_map(g, prefix, intr, pose=None, frame_index=0):
    """A duck-typed numpy map (reference field names) from golden arrays."""
    m = SimpleNamespace(frame_index=frame_index, pose=pose or Pose.identity(), intrinsics=intr)
    for k in PARAM_KEYS:
        v = np.asarray(g[prefix + k])
        setattr(m, k, v.astype(bool) if k == "active_mask" else v.astype(np.float64).copy())
    return m


def window_maps(g):
    intr = intr_from(g["intr"])
    maps = []
    i = 0
    while f"m{i}_base_depth" in g:
        maps.append(np_map(g, f"m{i}_", intr, pose_from(g[f"m{i}_pose"]), frame_index=i))
        i += 1
    return intr, maps


def rel_err(a, b, floor_frac=1e-3):
    """max |a-b| / max(|b|_inf * floor_frac, |b|) elementwise, reported as a max.

    Gradient parity bar (north_star): 1e-3 relative.  Entries whose reference
    magnitude is below ``floor_frac`` of the array's largest magnitude are
    measured against that floor (cancellation makes tiny entries' relative
    error meaningless for a sum reduced in a different order)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(float(np.abs(b).max()) if b.size else 0.0, 1e-300)
    den = np.maximum(np.abs(b), floor_frac * scale)
    return float((np.abs(a - b) / den).max()) if b.size else 0.0
