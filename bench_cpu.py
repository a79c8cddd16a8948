"""CPU legs of bench.py (its ``cpu_baseline`` leg and ``--impl reference``
arm): the reference algorithm timed on the box's host cores, in a process of
its own so the GPU arm's process never loads the CPU code.

    python bench_cpu.py map-ref   --config c4 [--target-s 15] [--threads T]
    python bench_cpu.py map-port  --config c4 [--target-s 15] [--threads T]
    python bench_cpu.py track-port --track c2|c4size [--iters K]

* ``map-ref``: the REAL reference (``raysplat`` from ``baseline/_ref``, its
  Numba kernels, loss upstream, chain rule and ``MapOptimizer``) through
  ``oracle/refwindow.py`` -- a window iteration with its views in a thread
  pool (raysplat/pipeline.py:212).  kind "reference".
* ``map-port``: the C restatement of the same kernels (``oracle/``) and the
  numpy Adam.  kind "port".
* ``track-port``: the oracle GICP (``oracle/track.py``, tracker.py:265-346
  with scipy's cKDTree) on the window-fitted local / global sets.

A mapping step is bounded: every view of the window (one per host thread, up
to the window size) over the first ``m`` window maps, ``m`` sized from a
one-map calibration step so a step takes about ``--target-s`` seconds, then
the optimizer step on those maps.  Each leg prints one JSON object.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

UNIT = "Gaussian-views/s"


def _config(name):
    from paper_2603_21055_b200 import scenes
    return {"c1": None, "c3": scenes.config_c3, "c4": scenes.config_c4,
            "c5": scenes.config_c5}[name]()


class _Step:
    """One bounded window-iteration sample on either CPU implementation."""

    def __init__(self, impl, wc, n_maps, threads):
        import numpy as np
        self.impl, self.wc, self.m = impl, wc, n_maps
        self.views = list(range(min(len(wc.frames), max(1, threads))))
        self.threads = threads
        self.hw = int(np.asarray(wc.params[0].active_mask).size)
        if impl == "reference":
            from oracle import refwindow as RW
            self.ref = RW.import_reference()
            self.ws = RW.WindowStep(self.ref, wc.intr, wc.poses[:n_maps], wc.params[:n_maps],
                                    wc.frames)
            self.ws.poses = wc.poses  # targets: every view of the window
        else:
            from types import SimpleNamespace

            from oracle import raster as O
            self.O = O
            self.maps = [SimpleNamespace(frame_index=i, pose=wc.poses[i], intrinsics=wc.intr,
                                         base_depth=np.array(p.base_depth, np.float64),
                                         delta=np.array(p.delta, np.float64),
                                         log_radius=np.array(p.log_radius, np.float64),
                                         opacity_logit=np.array(p.opacity_logit, np.float64),
                                         color=np.array(p.color, np.float64),
                                         active_mask=np.asarray(p.active_mask, bool))
                         for i, p in enumerate(wc.params[:n_maps])]
            self.opts = [O.Adam(m) for m in self.maps]
            O.lib()

    @property
    def gaussian_views(self):
        return self.m * self.hw * len(self.views)

    def run(self, pool):
        if self.impl == "reference":
            return self.ws.step(self.views, pool)
        wc, O = self.wc, self.O

        def one(v):
            fr = wc.frames[v]
            return O.mapping_loss(self.maps, fr.color, fr.depth, fr.valid_mask,
                                  wc.poses[v].rotation, wc.poses[v].translation, wc.intr,
                                  learnable_map="all")
        res = list(pool.map(one, self.views))
        for i, opt in enumerate(self.opts):
            acc = None
            for _, grads, _ in res:
                g = grads[i]
                if acc is None:
                    acc = g
                else:
                    acc.color += g.color
                    acc.radius += g.radius
                    acc.opacity_logit += g.opacity_logit
                    acc.delta += g.delta
            opt.step(acc)
        return sum(loss.total for loss, _, _ in res)


def map_leg(impl, cfg_name, target_s, threads, steps=1, warmup=1, log=None):
    """Calibrate on one map, size the sample to ~target_s per step, time it."""
    from concurrent.futures import ThreadPoolExecutor
    wc = _config(cfg_name)
    n_frames = len(wc.frames)
    with ThreadPoolExecutor(max_workers=threads) as pool:
        cal = _Step(impl, wc, 1, threads)
        t0 = time.perf_counter()
        cal.run(pool)   # also the JIT / library load
        t_cal = time.perf_counter() - t0
        t0 = time.perf_counter()
        cal.run(pool)
        t1 = time.perf_counter() - t0
        m = int(max(1, min(n_frames, round(target_s / max(t1, 1e-3)))))
        st = _Step(impl, wc, m, threads)
        for _ in range(max(0, warmup - 1)):
            st.run(pool)
        times = []
        for _ in range(steps):
            t0 = time.perf_counter()
            st.run(pool)
            times.append(time.perf_counter() - t0)
            if log:
                print(f"bench_cpu: {impl} step {len(times)}/{steps} {times[-1]:.2f} s",
                      file=sys.stderr, flush=True)
    gv = st.gaussian_views
    value = gv * len(times) / sum(times)
    what = ("the reference raysplat (baseline/_ref: Numba kernels, loss upstream, chain rule, "
            "MapOptimizer)" if impl == "reference" else
            "the oracle port (C restatement of the raysplat kernels + numpy Adam)")
    return {"value": value, "unit": UNIT, "cores": min(threads, len(st.views)),
            "kind": "reference" if impl == "reference" else "port",
            "times_s": times, "gaussian_views_per_step": gv,
            "sample": f"{cfg_name.upper()} window iteration sample on {what}: "
                      f"{len(st.views)} target views (one per thread) over the first {m} of "
                      f"{n_frames} window maps ({gv} Gaussian-views) + the optimizer step on "
                      f"those maps; {len(times)} step(s) of {sum(times) / len(times):.1f} s "
                      f"(calibration: 1 map {t1:.1f} s, first call {t_cal:.1f} s)"}


def ref_c1_leg(reps=3):
    """C1 (BASELINE config 0) through the reference's public API:
    mapping_loss(tau=0) = splat + splat_backward (mapper.py:106-157), median
    of ``reps`` after a JIT warm-up."""
    import numpy as np

    from oracle import refwindow as RW
    from paper_2603_21055_b200 import scenes
    ref = RW.import_reference()
    intr, frame, learn, target = scenes.config_c1()
    ri, maps = RW.ref_maps(ref, intr, [scenes.Pose.identity()], [learn])
    _, tmaps = RW.ref_maps(ref, intr, [scenes.Pose.identity()], [target])
    ident = ref.GEO.Pose.identity()
    t_out = ref.R.splat(tmaps, ident, ri)
    from raysplat.datasets import RgbdFrame
    tf = RgbdFrame(color=np.clip(t_out.color, 0, 1).astype(np.float32),
                   depth=t_out.depth.astype(np.float32), valid_mask=frame.valid_mask.copy(),
                   intrinsics=ri, timestamp=0.0, index=0)
    cfg = ref.M.MapperConfig(tau=0.0)
    ref.M.mapping_loss(maps, tf, ident, cfg)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        ref.M.mapping_loss(maps, tf, ident, cfg)
        times.append(time.perf_counter() - t0)
    t = sorted(times)[len(times) // 2]
    n = int(np.asarray(learn.active_mask).size)
    return {"value": n / t, "unit": UNIT, "cores": 1, "kind": "reference", "ms_per_call": t * 1e3,
            "sample": f"C1 160x120 mapping_loss (tau 0) fwd+bwd of {n} Gaussians, median of "
                      f"{reps}"}


def _track_sets(which):
    """Local (query) and global (reference frame) sets of a tracking config,
    fitted on the CPU with the oracle's window fit (D2)."""
    import numpy as np

    from oracle import track as OT
    from paper_2603_21055_b200 import scenes
    if which == "c2":
        intr, ref, qry, truth = scenes.config_c2()
    else:
        intr = scenes.Intrinsics(**scenes.C4_INTR)
        prims = scenes.room_scene(0)
        ref = scenes.render_frame(prims, scenes.Pose.identity(), intr, 0, depth_noise_rel=0.01)
        truth = scenes.se3_exp([0.01, -0.02, 0.015, 0.03, -0.01, 0.02])
        qry = scenes.render_frame(prims, truth, intr, 1, depth_noise_rel=0.01)
    out = []
    for fr in (ref, qry):
        _, c, rot, s, n = OT.window_fit(np.asarray(fr.depth), np.asarray(fr.valid_mask), intr.fx,
                                        intr.fy, intr.cx, intr.cy)
        out.append((c, OT.covariances(rot, s), n))
    return out


def track_leg(which, iters):
    import numpy as np

    from oracle import track as OT
    (gc, gcov, gn), (lc, lcov, _) = _track_sets(which)
    t0 = time.perf_counter()
    R, t, diag = OT.gicp_align(lc, lcov, gc, gcov, gn, np.eye(3), np.zeros(3), max_iters=iters,
                               eps=0.0)
    dt = time.perf_counter() - t0
    n_it = max(diag.iterations, 1)
    threads = os.environ.get("OPENBLAS_NUM_THREADS", "")
    return {"value": n_it / dt, "unit": "GN iters/s", "kind": "port",
            "cores": 1 if threads == "1" else len(os.sched_getaffinity(0)),
            "correspondences": int(len(lc)),
            "sample": f"oracle gicp_align (tracker.py:265-346 restated; scipy cKDTree exact NN, "
                      f"numpy normal equations) {n_it} GN iterations at {which}, "
                      f"{len(lc)} correspondences, {dt:.1f} s"}


def run_subprocess(argv, threads=None, timeout=900):
    """Run one leg in a child process; returns its JSON (or an error record)."""
    import subprocess
    env = dict(os.environ)
    if threads == 1:
        for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
            env[k] = "1"
    try:
        out = subprocess.run([sys.executable, os.path.abspath(__file__)] + argv, env=env,
                             capture_output=True, text=True, timeout=timeout)
        lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
        if out.returncode != 0 or not lines:
            return {"error": f"exit {out.returncode}: {out.stderr.strip()[-400:]}"}
        return json.loads(lines[-1])
    except Exception as exc:  # a CPU leg must not take the GPU line down
        return {"error": repr(exc)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("leg", choices=["map-ref", "map-port", "ref-c1", "track-port"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--track", default="c2")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--target-s", type=float, default=15.0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--steps", type=int, default=1)
    args = ap.parse_args()
    threads = args.threads or len(os.sched_getaffinity(0))
    if args.leg in ("map-ref", "map-port"):
        res = map_leg("reference" if args.leg == "map-ref" else "port", args.config,
                      args.target_s, threads, steps=args.steps)
    elif args.leg == "ref-c1":
        res = ref_c1_leg()
    else:
        res = track_leg(args.track, args.iters)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
