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


# ---------------------------------------------------------------- bench-config digests
# Compact, exact digests of one rendered view of a benched window (C3 / C4),
# computed the same way from the reference run (tests/golden/make_golden.py)
# and from this repo's GPU path (tests/test_bench_parity_gpu.py).

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def tile_digest(offsets, entry_frame, entry_pixel):
    """Per-tile order-sensitive 64-bit hash of the list entries (frame,
    pixel), tile t holding entries [offsets[t], offsets[t+1])."""
    offsets = np.asarray(offsets, dtype=np.int64)
    n = int(offsets[-1])
    key = (np.asarray(entry_frame, dtype=np.uint64) << np.uint64(32)) | \
        np.asarray(entry_pixel, dtype=np.uint64)
    pos = np.arange(n, dtype=np.int64) - np.repeat(offsets[:-1], np.diff(offsets))
    with np.errstate(over="ignore"):
        h = _splitmix(key ^ _splitmix(pos.astype(np.uint64)))
    out = np.zeros(len(offsets) - 1, dtype=np.uint64)
    nz = np.diff(offsets) > 0
    if n:
        out[nz] = np.add.reduceat(h, offsets[:-1][nz])
    return out


def sample_indices(n, k, seed):
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(n, size=min(k, n), replace=False))


def forced_params(params, lrs=(0.01, 0.005, 0.05, 0.0025), steps=3, seed=21):
    """The 'teacher-forced' window state of the bench fixtures: every
    learnable parameter moved by ``steps`` seeded steps of +-lr (the size of
    Adam's first steps, lr * g / (|g| + eps)) from the benched init, colour
    clipped to [0, 1], everything fp32-representable.  Groups: delta,
    log_radius, opacity_logit, colour (mapper.py:35-38)."""
    from copy import copy
    rng = np.random.default_rng(seed)
    out = []
    for p in params:
        q = copy(p)
        for name, lr in zip(("delta", "log_radius", "opacity_logit", "color"), lrs):
            v = np.asarray(getattr(p, name), dtype=np.float64)
            k = rng.integers(0, 2, size=(steps,) + v.shape).astype(np.float64) * 2.0 - 1.0
            nv = v + lr * k.sum(axis=0)
            if name == "color":
                nv = np.clip(nv, 0.0, 1.0)
            setattr(q, name, nv.astype(np.float32).astype(np.float64))
        out.append(q)
    return out
