"""CPU ORACLE for the tracking hot path -- test infrastructure, never the product.

Restates, in numpy (+ scipy's cKDTree for exact 1-NN, as the reference):
  * sym_eigh3_batch          /root/reference/pkg/src/raysplat/geometry.py:275-353
  * window fit (delta D2)    tracker.py:144-170 with the neighbour selection
                             replaced by the valid pixels of a 5x5 window
                             (self excluded, >= 4 of them)
  * gicp_align               tracker.py:265-346 (unchanged algorithm)
Pinned against tests/golden/track.npz and eig.npz, produced by the reference.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
from scipy.spatial import cKDTree

EIG_GAP_FALLBACK = 1e-8
EIGVAL_FLOOR_REL = 1e-6
PLANE_SCALES = (1.0, 1.0, 1e-3)
MIN_INLIERS = 10
MAX_STEP_HALVINGS = 5


def sym_eigh3_batch(mats):
    m = np.asarray(mats, dtype=np.float64)
    n = m.shape[0]
    rot = np.empty((n, 3, 3))
    vals = np.empty((n, 3))
    q = np.trace(m, axis1=1, axis2=2) / 3.0
    off = m[:, 0, 1] ** 2 + m[:, 0, 2] ** 2 + m[:, 1, 2] ** 2
    dd = m[:, [0, 1, 2], [0, 1, 2]] - q[:, None]
    p2 = (dd**2).sum(axis=1) + 2.0 * off
    scale = np.maximum(np.abs(m).max(axis=(1, 2)), 1e-300)
    iso = p2 <= (1e-14 * scale) ** 2
    vals[iso] = q[iso, None]
    rot[iso] = np.eye(3)
    gen = ~iso
    if gen.any():
        mg, qg = m[gen], q[gen]
        p = np.sqrt(p2[gen] / 6.0)
        b = (mg - qg[:, None, None] * np.eye(3)) / p[:, None, None]
        phi = np.arccos(np.clip(np.linalg.det(b) / 2.0, -1.0, 1.0)) / 3.0
        e1 = qg + 2.0 * p * np.cos(phi)
        e3 = qg + 2.0 * p * np.cos(phi + 2.0 * np.pi / 3.0)
        e2 = 3.0 * qg - e1 - e3
        ev = np.stack([e1, e2, e3], axis=1)
        ok = np.minimum(e1 - e2, e2 - e3) / scale[gen] > EIG_GAP_FALLBACK
        r = np.empty((int(gen.sum()), 3, 3))
        if ok.any():
            r[ok] = _projector(mg[ok], ev[ok])
        if (~ok).any():
            w, vec = np.linalg.eigh(mg[~ok])
            ev[~ok] = w[:, ::-1]
            r[~ok] = vec[:, :, ::-1]
        vals[gen] = ev
        rot[gen] = r
    flip = np.linalg.det(rot) < 0
    rot[flip, :, 2] *= -1.0
    return rot, vals


def _projector(m, ev):
    eye = np.eye(3)

    def col(a):
        idx = np.argmax(np.linalg.norm(a, axis=1), axis=1)
        c = a[np.arange(len(a)), :, idx]
        return c / np.linalg.norm(c, axis=1, keepdims=True)

    m1 = m - ev[:, 0, None, None] * eye
    m2 = m - ev[:, 1, None, None] * eye
    m3 = m - ev[:, 2, None, None] * eye
    v1 = col(m2 @ m3)
    v3 = col(m1 @ m2)
    v3 = v3 - (v3 * v1).sum(axis=1, keepdims=True) * v1
    v3 /= np.linalg.norm(v3, axis=1, keepdims=True)
    return np.stack([v1, np.cross(v3, v1), v3], axis=2)


def _normalize(scales, mode):
    if mode == "ellipse":
        return scales / np.linalg.norm(scales, axis=1, keepdims=True)
    if mode == "plane":
        return np.broadcast_to(np.array(PLANE_SCALES), scales.shape).copy()
    return scales


def window_fit(depth, mask, fx, fy, cx, cy, stride=1, win=5, k_min=4, scale_mode="ellipse"):
    """Local geometry Gaussians of one frame with the window neighbourhood.
    Returns (pixel index, centers, rotations, scales, normals) in row-major
    pixel order of the sampled valid pixels that have >= k_min neighbours."""
    depth = np.asarray(depth)
    valid = np.asarray(mask, dtype=bool)
    h, w = depth.shape
    vs, us = np.nonzero(valid)
    z = depth[vs, us].astype(np.float64)
    pts = np.zeros((h, w, 3))
    pts[vs, us] = np.stack([(us - cx) / fx * z, (vs - cy) / fy * z, z], axis=1)
    r = win // 2
    # gather window neighbours with array shifts
    offs = [(dv, du) for dv in range(-r, r + 1) for du in range(-r, r + 1) if (dv, du) != (0, 0)]
    pad_v = np.zeros((h + 2 * r, w + 2 * r), dtype=bool)
    pad_v[r:r + h, r:r + w] = valid
    pad_p = np.zeros((h + 2 * r, w + 2 * r, 3))
    pad_p[r:r + h, r:r + w] = pts
    grid = np.zeros((h, w), dtype=bool)
    grid[::stride, ::stride] = True
    cand = valid & grid
    cv, cu = np.nonzero(cand)
    nb_ok = np.stack([pad_v[cv + r + dv, cu + r + du] for dv, du in offs], axis=1)
    nb_pt = np.stack([pad_p[cv + r + dv, cu + r + du] for dv, du in offs], axis=1)
    k = nb_ok.sum(axis=1)
    keep = k >= k_min
    cv, cu, nb_ok, nb_pt, k = cv[keep], cu[keep], nb_ok[keep], nb_pt[keep], k[keep]
    wts = nb_ok[..., None].astype(np.float64)
    mean = (nb_pt * wts).sum(axis=1) / k[:, None]
    diff = (nb_pt - mean[:, None, :]) * wts
    cov = np.einsum("nki,nkj->nij", diff, diff) / k[:, None, None]
    centers = pts[cv, cu]
    rot, vals = sym_eigh3_batch(cov)
    vals = np.maximum(vals, EIGVAL_FLOOR_REL * vals[:, :1])
    scales = _normalize(np.sqrt(vals), scale_mode)
    normals = rot[:, :, 2].copy()
    flip = np.einsum("ni,ni->n", normals, -centers) < 0.0
    normals[flip] *= -1.0
    rot[flip, :, 2] *= -1.0
    rot[flip, :, 1] *= -1.0
    return cv * w + cu, centers, rot, scales, normals


def covariances(rot, scales):
    return np.einsum("nij,nj,nkj->nik", rot, scales**2, rot)


def se3_exp(twist):
    twist = np.asarray(twist, dtype=np.float64).reshape(6)
    w, v = twist[:3], twist[3:]
    th = np.linalg.norm(w)
    wx = np.array([[0.0, -w[2], w[1]], [w[2], 0.0, -w[0]], [-w[1], w[0], 0.0]])
    if th < 1e-8:
        r = np.eye(3) + wx + 0.5 * (wx @ wx)
        jl = np.eye(3) + 0.5 * wx + (wx @ wx) / 6.0
    else:
        r = np.eye(3) + np.sin(th) / th * wx + (1.0 - np.cos(th)) / (th * th) * (wx @ wx)
        t2 = th * th
        jl = np.eye(3) + (1.0 - np.cos(th)) / t2 * wx + (th - np.sin(th)) / (t2 * th) * (wx @ wx)
    return r, jl @ v


def _skew(p):
    out = np.zeros(p.shape[:-1] + (3, 3))
    x, y, z = p[..., 0], p[..., 1], p[..., 2]
    out[..., 0, 1] = -z
    out[..., 0, 2] = y
    out[..., 1, 0] = z
    out[..., 1, 2] = -x
    out[..., 2, 0] = -y
    out[..., 2, 1] = x
    return out


@dataclass
class Diag:
    iterations: int = 0
    final_cost: float = float("nan")
    inlier_count: int = 0
    converged: bool = False
    failed: bool = False
    cost_pairs: list = field(default_factory=list)
    accepted_first: np.ndarray | None = None
    systems: list = field(default_factory=list)


def gicp_align(l_centers, l_cov, g_centers, g_cov, g_normals, init_rot, init_t, max_iters=30,
               dist_max=0.2, eps=1e-5, metric_mode="point2surf"):
    """tracker.py:265-346 restated over plain arrays (poses as (R, t))."""
    tree = cKDTree(g_centers)
    diag = Diag()
    R, t = np.asarray(init_rot, dtype=np.float64), np.asarray(init_t, dtype=np.float64)
    R0, t0 = R.copy(), t.copy()
    for it in range(max_iters):
        pts = l_centers @ R.T + t
        dist, j = tree.query(pts, k=1)
        b = g_centers[j]
        d = b - pts
        metric = np.abs(np.einsum("ni,ni->n", g_normals[j], d)) if metric_mode == "point2surf" \
            else dist
        acc = metric < dist_max
        n_acc = int(acc.sum())
        diag.inlier_count = n_acc
        if it == 0:
            diag.accepted_first = acc.copy()
        if n_acc < MIN_INLIERS:
            diag.failed = True
            return R0, t0, diag
        c_comb = g_cov[j[acc]] + np.einsum("ij,njk,lk->nil", R, l_cov[acc], R)
        w = np.linalg.inv(c_comb)
        a_w, b_w = l_centers[acc], b[acc]

        def cost_at(Rc, tc):
            res = b_w - (a_w @ Rc.T + tc)
            return float(np.einsum("ni,nij,nj->", res, w, res))

        cost_before = cost_at(R, t)
        p_acc = pts[acc]
        jac = np.concatenate([_skew(p_acc), -np.broadcast_to(np.eye(3), (n_acc, 3, 3))], axis=2)
        h = np.einsum("nij,nik,nkl->jl", jac, w, jac)
        g = np.einsum("nij,nik,nk->j", jac, w, d[acc])
        diag.systems.append((h, g, cost_before, n_acc))
        try:
            xi = np.linalg.solve(h, -g)
        except np.linalg.LinAlgError:
            xi = np.linalg.lstsq(h, -g, rcond=None)[0]

        def cand(x):
            dr, dt = se3_exp(x)
            return dr @ R, dr @ t + dt

        Rc, tc = cand(xi)
        halv = 0
        while cost_at(Rc, tc) > cost_before and halv < MAX_STEP_HALVINGS:
            xi = 0.5 * xi
            Rc, tc = cand(xi)
            halv += 1
        cost_after = cost_at(Rc, tc)
        if cost_after > cost_before:
            diag.final_cost = cost_before
            break
        R, t = Rc, tc
        diag.iterations += 1
        diag.final_cost = cost_after
        diag.cost_pairs.append((cost_before, cost_after))
        if np.linalg.norm(xi) < eps:
            diag.converged = True
            break
    return R, t, diag


# ---------------------------------------------------------------------------
# Render-based pose initialiser (tracker.py:354-426), restated on the oracle
# rasterizer: L1 photometric + weighted, valid-masked L1 depth residuals, a
# central-difference Jacobian through the renderer (step 1e-4 on each twist
# component, applied on the left), three IRLS solves per linearisation
# (weights 1 / max(|predicted residual|, 1e-3), least squares), up to 5 step
# halvings, a coverage gate (alpha > 0.5 on >= 30 % of the pixels).

def _compose(ra, ta, rb, tb):
    return ra @ rb, ra @ tb + ta


def init_pose_render(tcolor, tdepth, tmask, prev_map, init_rot, init_t, intr, iters=10,
                     depth_weight=4.0, coverage_min=0.3):
    from . import raster as R
    tc = np.asarray(tcolor, dtype=np.float64)
    td = np.asarray(tdepth, dtype=np.float64)
    m = np.asarray(tmask, dtype=np.float64)

    def resid(rot, t):
        out = R.splat([prev_map], rot, t, intr)
        return np.concatenate([(out.color - tc).ravel(),
                               (depth_weight * m * (out.depth - td)).ravel()])

    cover = float((R.splat([prev_map], init_rot, init_t, intr).alpha > 0.5).mean())
    if cover < coverage_min:
        return init_rot, init_t, False
    rot, t = np.asarray(init_rot, dtype=np.float64), np.asarray(init_t, dtype=np.float64)
    step = 1e-4
    r = resid(rot, t)
    for _ in range(iters):
        jac = np.empty((r.size, 6))
        for k in range(6):
            tw = np.zeros(6)
            tw[k] = step
            ep, em = se3_exp(tw), se3_exp(-tw)
            jac[:, k] = (resid(*_compose(*ep, rot, t)) - resid(*_compose(*em, rot, t))) / (2 * step)
        xi = np.zeros(6)
        for _irls in range(3):
            wts = 1.0 / np.maximum(np.abs(r + jac @ xi), 1e-3)
            xi = np.linalg.lstsq(jac.T @ (jac * wts[:, None]), -(jac.T @ (wts * r)), rcond=None)[0]
        cost = float(np.abs(r).sum())
        cand = _compose(*se3_exp(xi), rot, t)
        rc = resid(*cand)
        halvings = 0
        while float(np.abs(rc).sum()) > cost and halvings < 5:
            xi = 0.5 * xi
            cand = _compose(*se3_exp(xi), rot, t)
            rc = resid(*cand)
            halvings += 1
        if float(np.abs(rc).sum()) > cost:
            break
        (rot, t), r = cand, rc
        if np.linalg.norm(xi) < 1e-7:
            break
    return rot, t, True


class VoxelSet:
    """Cell gating of GlobalGeomSet.insert (tracker.py:101-122) restated: at
    most one member per cell floor(c / voxel), first come first served in row
    order within a batch."""

    def __init__(self, voxel):
        self.voxel = voxel
        self.cells = set()

    def gate(self, centers):
        keys = np.floor(np.asarray(centers, dtype=np.float64) / self.voxel).astype(np.int64)
        keep = np.zeros(len(keys), dtype=bool)
        for i, k in enumerate(map(tuple, keys)):
            if k not in self.cells:
                self.cells.add(k)
                keep[i] = True
        return keep


def inpaint_depth(depth, valid_mask, max_iters=200, tol=1e-5):
    """datasets.py:368-398 restated: nearest-valid seeding (scipy's Euclidean
    distance transform, the reference's call) then Jacobi sweeps of the
    Laplace equation on the holes with edge-replicated borders, stopping
    after the first sweep whose largest update is below ``tol``."""
    from scipy import ndimage
    z = np.asarray(depth, dtype=np.float64)
    ok = np.asarray(valid_mask, dtype=bool) & (z > 0)
    if not ok.any():
        raise ValueError("cannot inpaint a frame with no valid depth")
    if ok.all():
        return z.copy()
    _, (iy, ix) = ndimage.distance_transform_edt(~ok, return_indices=True)
    cur = z[iy, ix]
    cur[ok] = z[ok]
    holes = ~ok
    for _ in range(max_iters):
        e = np.pad(cur, 1, mode="edge")
        nxt = 0.25 * (e[:-2, 1:-1] + e[2:, 1:-1] + e[1:-1, :-2] + e[1:-1, 2:])
        step = np.abs(nxt[holes] - cur[holes]).max()
        cur[holes] = nxt[holes]
        if step < tol:
            break
    return cur
