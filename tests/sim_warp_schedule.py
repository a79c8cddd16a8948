"""CPU replay of the compositing kernels' warp schedule on the oracle's tile
lists (design evidence for DESIGN.md K4/K5; not collected by pytest).

For every 8x4 sub-tile of a sample of C4 tiles it counts the contributions
(pixel, Gaussian passes, before termination) and the warp iterations a warp
needs when (a) one window of 33..64 useful entries is composited at a time
(the warp waits for the window's busiest lane) or (b) lanes consume a ring
of R windows at their own pace.  busy lanes per iteration = contributions /
iterations.

    python tests/sim_warp_schedule.py [tile_step]
"""
import os
import sys
from types import SimpleNamespace

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import raster as O  # noqa: E402
from paper_2603_21055_b200 import scenes  # noqa: E402


def windows(cov, contrib, term):
    useful = np.nonzero(cov.any(1))[0]
    chunk_of = useful // 32
    out, i, nu = [], 0, len(useful)
    while i < nu:
        n, j = 0, i
        while j < nu and n <= 32:
            c, k = chunk_of[j], j
            while k < nu and chunk_of[k] == c:
                k += 1
            n += k - j
            j = k
        sel = useful[i:j]
        alive = term >= sel[0]
        if not alive.any():
            break
        out.append(contrib[sel].sum(0) * alive)
        i = j
    return out


def ring_iters(wins, ring):
    rem = [w.copy() for w in wins]
    nw = len(wins)
    lane_w = np.zeros(32, dtype=np.int64)
    head = min(ring, nw)
    it = 0
    while True:
        for L in range(32):
            while lane_w[L] < head and rem[lane_w[L]][L] == 0:
                lane_w[L] += 1
        while head < nw and (lane_w >= head - ring + 1).all():
            head += 1
            for L in range(32):
                while lane_w[L] < head and rem[lane_w[L]][L] == 0:
                    lane_w[L] += 1
        act = lane_w < head
        if not act.any():
            return it
        it += 1
        for L in np.nonzero(act)[0]:
            rem[lane_w[L]][L] -= 1


def main():
    step = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    wc = scenes.config_c4("cpu")
    maps = [SimpleNamespace(frame_index=i, pose=wc.poses[i], intrinsics=wc.intr,
                            base_depth=p.base_depth, delta=p.delta, log_radius=p.log_radius,
                            opacity_logit=p.opacity_logit, color=p.color,
                            active_mask=p.active_mask) for i, p in enumerate(wc.params)]
    v = 3
    b = O.prepare(maps, wc.poses[v].rotation, wc.poses[v].translation, wc.intr, learnable="all")
    off, lst = O.tile_lists(b)
    W, H = wc.intr.width, wc.intr.height
    ntx = (W + 15) // 16
    rings = (1, 2, 4, 8, 16, 10 ** 9)
    tot = {r: 0 for r in rings}
    contrib_total = 0
    for t in range(0, len(off) - 1, step):
        ids = lst[off[t]:off[t + 1]]
        if len(ids) == 0:
            continue
        ty, tx = divmod(t, ntx)
        U, V, S, OP = b.u0[ids], b.v0[ids], b.sigma[ids], b.opacity[ids]
        for w in range(8):
            px = tx * 16 + (w & 1) * 8 + np.arange(32) % 8
            py = ty * 16 + (w >> 1) * 4 + np.arange(32) // 8
            valid = (px < W) & (py < H)
            dx, dy = U[:, None] - px[None, :], V[:, None] - py[None, :]
            d2 = dx * dx + dy * dy
            cov = (d2 <= 9 * S[:, None] ** 2) & valid[None, :]
            a = np.where(cov, np.minimum(OP[:, None] * np.exp(-0.5 * d2 / S[:, None] ** 2), 0.999),
                         0.0)
            after = np.cumprod(1 - a, axis=0) < 1e-4
            term = np.where(after.any(0), after.argmax(0), len(ids))
            contrib = cov & (np.arange(len(ids))[:, None] <= term[None, :])
            contrib_total += int(contrib.sum())
            wins = windows(cov, contrib, term)
            for r in rings:
                tot[r] += sum(int(x.max()) for x in wins) if r == 1 else ring_iters(wins, r)
    for r in rings:
        name = "one window" if r == 1 else ("unbounded ring" if r > 100 else f"ring of {r}")
        print(f"{name:16s} busy lanes / iteration {contrib_total / max(tot[r], 1):5.1f}")


if __name__ == "__main__":
    main()
