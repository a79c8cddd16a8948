"""Benchmark of the graded hot path (BASELINE.json metric: mapping fwd+bwd
Gaussians/s at 1200x680, 8-keyframe window; tracking GN iterations/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one window iteration of configuration C4: every keyframe's view is
rendered (K1-K4 with the fused tau=0 L1 loss), back-propagated (K5) onto all
6.5 M pixel-aligned Gaussians, the gradients are exchanged over ranks (NCCL
reduce-scatter by frame block, Adam per block, all-gather) and Adam updates
the window.  Views are sharded over ranks; the window is fixed, so total work
is fixed (``scaling`` = "strong").  Inputs are synthetic (seeded room scene,
DESIGN.md).  ``--gpus N`` without a torchrun environment re-executes itself
under torch.distributed.run with N ranks.

``--impl reference`` times the reference itself (the raysplat package from
baseline/_ref, its Numba kernels and MapOptimizer) on the host cores, rank 0
only; the CPU legs of our line (the reference, the oracle port, tracking)
run in child processes (bench_cpu.py).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "mapping fwd+bwd Gaussians/s (C4 1200x680, 8-keyframe window)"
METRICS = {"c3": "mapping fwd+bwd Gaussians/s (C3 640x480, 8-keyframe window)",
           "c4": METRIC,
           "c5": "mapping fwd+bwd Gaussians/s (C5 1200x680, 32-keyframe window)"}
UNIT = "Gaussian-views/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=["c3", "c4", "c5"])
    ap.add_argument("--tau", type=float, default=0.0,
                    help="SSIM weight of the objective (BASELINE C4: colour+depth L1, tau 0)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-track", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--launch-check", action="store_true",
                    help="only start the ranks, join a process group (gloo without GPUs) and "
                         "report them (tests the --gpus N launch)")
    return ap.parse_args()


def launch_check(args):
    """--launch-check: the rank launch of --gpus N without any GPU work."""
    import torch
    import torch.distributed as dist
    rank, world, _ = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
        t = torch.tensor([rank + 1.0])
        dist.all_reduce(t)
        assert dist.get_world_size() == args.gpus and int(t.item()) == world * (world + 1) // 2
    if rank == 0:
        print(json.dumps({"launch_check": True, "world_size": world}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def make_config(name, device):
    from paper_2603_21055_b200 import scenes
    if name == "c3":
        return scenes.config_c3(device=device)
    if name == "c5":
        return scenes.config_c5(device=device)
    return scenes.config_c4(device=device)


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max((float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ CPU legs


def workload_config(cfg_name, tau, world):
    """The ``config`` object of both arms' lines (identical by construction)."""
    from paper_2603_21055_b200 import scenes
    intr = {"c3": scenes.C3_INTR, "c4": scenes.C4_INTR, "c5": scenes.C4_INTR}[cfg_name]
    n_views = 32 if cfg_name == "c5" else 8
    w, h = intr["width"], intr["height"]
    return {"workload": f"{cfg_name.upper()}: {w}x{h}, {n_views}-keyframe window, all learnable, "
                        f"tau={tau:g} L1 colour+depth{' + SSIM' if tau else ''}, Adam",
            "gaussians": n_views * w * h, "views_per_step": n_views,
            "parallelism": (f"views sharded over {world} GPU(s); gradient reduce-scatter by "
                            "frame block, Adam per block, parameter all-gather (NCCL)"
                            if world > 1 else "1 GPU"),
            "l2": "inputs larger than L2 (params 183 MB + records ~350 MB/view at C4)"}


def run_reference(args):
    """The reference arm: the reference's own CPU implementation -- the
    raysplat package itself (``baseline/_ref``: its Numba kernels, loss,
    chain rule and MapOptimizer, bench_cpu.py / oracle/refwindow.py) -- on the
    box's host cores, on this arm's config, metric and unit.  A step is a
    bounded sample of the window iteration: every view (one per host thread)
    over the first m window maps, m sized so a step takes ~``150 / K`` s, then
    the reference Adam on those maps.  Under torchrun rank 0 alone runs; the
    other ranks exit."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import bench_cpu
    threads = len(os.sched_getaffinity(0))
    k, w = max(1, args.steps), max(0, args.warmup)
    target = max(2.0, min(20.0, 150.0 / k))
    cb = bench_cpu.map_leg("reference", args.config, target, threads, steps=k, warmup=w, log=True)
    value = cb["value"]
    timed = cb.pop("times_s")
    line = {"metric": METRICS[args.config], "value": value, "unit": UNIT, "n_gpus": world,
            "steps": k, "warmup": w, "ms_per_step": 1e3 * sum(timed) / k,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.config, args.tau, world),
            "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2603_21055_b200.mapper import MapperConfig, WindowMapper

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: {world} ranks but {torch.cuda.device_count()} visible GPU(s)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        assert dist.get_world_size() == args.gpus
        print(f"bench.py: rank {dist.get_rank()}/{dist.get_world_size()} on cuda:{local} "
              f"({torch.cuda.get_device_name(dev)}), NCCL {torch.cuda.nccl.version()}",
              file=sys.stderr, flush=True)
    wc = make_config(args.config, dev)
    views = list(range(rank, len(wc.poses), world))
    wm = WindowMapper(wc.frames, wc.poses, wc.intr, wc.params, MapperConfig(tau=args.tau),
                      views=views, device=dev)
    if os.environ.get("SGAD_PIPELINE") == "0":  # A/B: no prepare/composite overlap
        wm.pipelined = False
    if os.environ.get("SGAD_FUSE") == "1":  # A/B: forward + backward as one kernel
        wm.fuse_fwd_bwd = True
    # the window step as one CUDA graph (captured at the first warm-up step);
    # SGAD_GRAPH=0: launched eagerly (A/B).  Multi-rank runs stay eager: the
    # NCCL exchange is not captured (no multi-GPU box to validate it here)
    wm.use_graph = world == 1 and os.environ.get("SGAD_GRAPH", "1") != "0"
    n_g = wm.n_gaussians
    n_views_total = len(wc.poses)

    # per-view kernel timing: CUDA events recorded by the window engine on the
    # streams the kernels run on (prepare on its side stream, compositing on
    # the main stream)
    stream = torch.cuda.current_stream()
    timing = []

    for _ in range(args.warmup):
        wm.step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    from paper_2603_21055_b200 import _native as N
    sampler = ClockSampler(local)
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    with sampler:
        torch.cuda.synchronize()
        start.record(stream)
        for _ in range(args.steps):
            wm.step(timing=None if wm.use_graph else timing)
        stop.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # per-kernel breakdown and launch count: two eager steps with CUDA events
    # on the kernels' own streams (a graph replay has no per-view events and
    # does not pass through the library's launch counter)
    launches0 = N.launch_count()
    for _ in range(2):
        wm.step(timing=timing)
    torch.cuda.synchronize()
    launches_per_step = (N.launch_count() - launches0) / 2
    launches = int(launches_per_step * args.steps)
    ms = start.elapsed_time(stop)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ms_step = ms / args.steps
    value = n_g * n_views_total * args.steps / (ms / 1e3)

    # roofline of the compositing kernels (SURVEY 8d algorithmic bytes)
    hw = wm.HW

    counts = wm.counts()  # per view (survivors, tile pairs): the same every step (fixed window)

    def kstats(kind, extra_surv, both=False):
        lst = [t for t in timing if t[0] == kind]
        tot_ms = sum(a.elapsed_time(b) for _, a, b, _ in lst)
        per = (lambda ns, npairs: 72 * npairs + 40 * hw + 32 * ns) if both else \
            (lambda ns, npairs: 36 * npairs + 20 * hw + (32 * ns if extra_surv else 0))
        tot_bytes = sum(per(*counts[v]) for _, _, _, v in lst)
        return tot_ms, tot_bytes, len(lst)

    f_ms, f_bytes, f_n = kstats("fwd", False)
    b_ms, b_bytes, b_n = kstats("bwd", True)
    fb_ms, fb_bytes, fb_n = kstats("fb", False, both=True)
    p_ms, _, p_n = kstats("prep", False)
    peak, peak_kind = load_peaks()
    if fb_n:  # forward + loss + backward in one kernel (tau = 0)
        dom = ("k_forward_backward", fb_ms, fb_bytes, fb_n)
    else:
        dom = ("k_backward", b_ms, b_bytes, b_n) if b_ms >= f_ms else \
            ("k_forward", f_ms, f_bytes, f_n)
    achieved = dom[2] / dom[3] / (dom[1] / dom[3] / 1e3) / 1e9
    mean_ns = float(np.mean([c[0] for c in counts.values()])) if counts else 0.0
    mean_np = float(np.mean([c[1] for c in counts.values()])) if counts else 0.0
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f)["dram_bytes_per_launch"].get(dom[0])
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": dom[0], "achieved": achieved, "peak": peak,
                "peak_source": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_source": "profiles/traffic.json (ncu --set full)",
                "launch_ms": dom[1] / dom[3],
                "bytes_per_launch": dom[2] / dom[3],
                "forward_ms_per_view": f_ms / max(f_n, 1) if f_n else None,
                "backward_ms_per_view": b_ms / max(b_n, 1) if b_n else None,
                "forward_backward_ms_per_view": fb_ms / fb_n if fb_n else None,
                "prepare_ms_per_view": p_ms / max(p_n, 1),
                "prepare_overlapped": bool(wm.pipelined),
                "mean_survivors_per_view": mean_ns, "mean_pairs_per_view": mean_np}
    # the whole window iteration against the same peak (per view
    # 52 N + 80 P + 57 HW bytes, N = the window's Gaussians; + 168 N for Adam)
    # (this rank's views, scaled to the window's: all ranks' views per step)
    b_iter = (n_views_total / max(len(counts), 1) *
              sum(52 * n_g + 80 * counts[v][1] + 57 * hw for v in counts) + 168 * n_g)
    roofline["step"] = {"bytes": b_iter, "achieved_gbs": b_iter / (ms_step / 1e3) / 1e9,
                        "frac": b_iter / (ms_step / 1e3) / 1e9 / peak}

    # e2e through the public API with host buffers (targets up, loss down; and
    # the conservative variant with the parameters up and down every step)
    e2e = e2e_params = None
    if not args.no_e2e:
        e2e = measure_e2e(wm, args, dev, world)
        e2e_params = measure_e2e(wm, args, dev, world, with_params=True)

    ssim_line = None
    if rank == 0:
        try:
            ssim_line = bench_ssim(dev)
        except Exception as exc:
            ssim_line = {"error": repr(exc)}

    track = track_c2 = None
    if not args.no_track and rank == 0:
        try:
            track = bench_tracking(dev, "c4size")
        except Exception as exc:  # tracking is the secondary metric
            track = {"error": repr(exc)}
        try:
            track_c2 = bench_tracking(dev, "c2")
        except Exception as exc:
            track_c2 = {"error": repr(exc)}
        try:
            track["rendered_geometry"] = bench_tracking_rendered(dev, wc)
        except Exception as exc:
            track["rendered_geometry"] = {"error": repr(exc)}
        try:
            track["render_init"] = bench_render_init(dev)
        except Exception as exc:
            track["render_init"] = {"error": repr(exc)}

    cpu = cpu_port = cpu_c1 = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the reference itself (kind "reference") and the oracle port beside it,
        # each in a process of its own (bench_cpu.py)
        import bench_cpu
        cpu = bench_cpu.run_subprocess(["map-ref", "--config", args.config, "--target-s", "15"])
        cpu_port = bench_cpu.run_subprocess(["map-port", "--config", args.config,
                                             "--target-s", "15"])
        cpu_c1 = bench_cpu.run_subprocess(["ref-c1"])
        for c in (cpu, cpu_port):
            c.pop("times_s", None)
        if track is not None and "error" not in track:
            track["cpu_baseline"] = bench_cpu.run_subprocess(
                ["track-port", "--track", "c4size", "--iters", "2"], threads=1)
        if track_c2 is not None and "error" not in track_c2:
            track_c2["cpu_baseline"] = bench_cpu.run_subprocess(
                ["track-port", "--track", "c2", "--iters", "5"], threads=1)
            track_c2["cpu_baseline_all_cores"] = bench_cpu.run_subprocess(
                ["track-port", "--track", "c2", "--iters", "5"])

    if rank == 0:
        line = {"metric": METRICS[args.config], "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64 composite / fp32 params", "data": "synthetic",
                "config": workload_config(args.config, args.tau, world),
                "window_iters_per_s": 1e3 / ms_step,
                "keyframes_per_s": n_views_total * 1e3 / ms_step / 100.0,
                "roofline": roofline, "cpu_baseline": cpu, "cpu_baseline_port": cpu_port,
                "cpu_reference_c1": cpu_c1, "e2e": e2e, "e2e_with_params": e2e_params,
                "gpu_launches": launches,
                "gpu_launches_note": (f"{launches_per_step:.0f} libsgad kernels per step"
                                      + (" (replayed from one CUDA graph per step)"
                                         if wm.use_graph else "")),
                "clocks": sampler.summary(), "tracking": track, "tracking_c2": track_c2,
                "ssim_term": ssim_line}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def measure_e2e(wm, args, dev, world, with_params=False):
    """Same metric through the reference-facing call with HOST buffers: every
    step uploads this rank's targets (the step's inputs: colour, depth and
    valid mask of every view it renders) from pinned host memory and reads
    the loss (the step's result) back into pinned host memory; the window
    parameters are the model state and stay resident in HBM.  With
    ``with_params`` every step also uploads the parameters and reads the
    updated ones back (a host-resident map, the conservative variant).  The
    copies run on a copy stream: the parameters (needed by every view)
    before any compositing; each view's target while earlier views
    composite; the parameter read-back of step s (from a device snapshot)
    while step s+1 runs.  All of them are inside the timed region."""
    import torch
    import torch.distributed as dist
    host_params = wm.planes.cpu().pin_memory()
    host_out = torch.empty_like(host_params).pin_memory()
    host_loss = torch.empty((), dtype=torch.float64).pin_memory()
    snap = torch.empty_like(wm.planes)
    vs = list(wm.views)
    host_tc = wm.tcolor[vs].cpu().pin_memory()
    host_td = wm.tdepth[vs].cpu().pin_memory()
    host_tm = wm.tmask[vs].cpu().pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in (host_tc, host_td, host_tm))
    d2h = host_loss.element_size()
    if with_params:
        h2d += host_params.numel() * host_params.element_size()
        d2h += host_out.numel() * host_out.element_size()
    steps = max(2, args.steps // 2)
    main = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)   # host -> device
    back = torch.cuda.Stream(dev)   # device -> host (runs beside the next step's uploads)
    state = {"d2h_done": None, "step_done": None}

    def one():
        with torch.cuda.stream(copy):
            if state["step_done"] is not None:  # the previous step no longer reads them
                copy.wait_event(state["step_done"])
            if with_params:
                wm.planes.copy_(host_params, non_blocking=True)
            params_ready = torch.cuda.Event()
            params_ready.record(copy)
            ready = {}
            for j, v in enumerate(vs):
                wm.tcolor[v].copy_(host_tc[j], non_blocking=True)
                wm.tdepth[v].copy_(host_td[j], non_blocking=True)
                wm.tmask[v].copy_(host_tm[j], non_blocking=True)
                ready[v] = torch.cuda.Event()
                ready[v].record(copy)
        main.wait_event(params_ready)
        loss = wm.step(target_ready=ready)
        if with_params:
            if state["d2h_done"] is not None:  # the snapshot is free again
                main.wait_event(state["d2h_done"])
            snap.copy_(wm.planes)
        host_loss.copy_(loss, non_blocking=True)
        done = torch.cuda.Event()
        done.record(main)
        state["step_done"] = done
        if with_params:
            with torch.cuda.stream(back):
                back.wait_event(done)
                host_out.copy_(snap, non_blocking=True)
                d = torch.cuda.Event()
                d.record(back)
                state["d2h_done"] = d

    def one_targets():
        # the public call: targets uploaded as part of the step (replayed
        # from one CUDA graph with use_graph), the loss read back
        loss = wm.step_with_targets(host_tc, host_td, host_tm)
        host_loss.copy_(loss, non_blocking=True)

    run = one if with_params else one_targets
    run()
    run()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for _ in range(steps):
        run()
    main.wait_stream(back)  # the last read-back is inside the timed region
    stop.record()
    torch.cuda.synchronize()
    ms = start.elapsed_time(stop)
    assert math.isfinite(float(host_loss))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"value": wm.n_gaussians * wm.F * steps / (ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": ms / steps, "steps": steps,
            "copies": ("pinned host buffers: uploads on a copy stream (parameters before "
                       "the step's compositing, targets per view overlapping it), the "
                       "read-back of parameters + loss on a second stream overlapping the "
                       "next step") if with_params else
                      ("WindowMapper.step_with_targets: every step's targets (colour, depth, "
                       "mask of each view) uploaded from pinned host buffers on a copy "
                       "stream, each view compositing once its target has arrived, the "
                       "loss read back; uploads + step replayed from one CUDA graph when "
                       "use_graph; the window parameters (model state) stay in HBM")}


def bench_ssim(dev, reps=20):
    """SSIM term (tau != 0 objective) at C4 size: sgad_ssim with the fused
    colour upstream on a 1200x680x3 pair (fp64 render, fp32 target), CUDA
    events on the launching stream.  Algorithmic bytes per call: images read
    twice (8 + 4 B per value), three fp64 maps written and read (48 B), the
    upstream written (8 B) = 72 B per pixel-channel."""
    import torch
    from paper_2603_21055_b200.ssim import ssim_sum, workspace_bytes
    h, w, c = 680, 1200, 3
    g = torch.Generator(device=dev).manual_seed(5)
    a = torch.rand((h, w, c), dtype=torch.float64, device=dev, generator=g)
    b = torch.rand((h, w, c), dtype=torch.float32, device=dev, generator=g)
    acc = torch.zeros((), dtype=torch.float64, device=dev)
    up = torch.empty_like(a)
    ws = torch.empty(workspace_bytes(h, w, c) // 8, dtype=torch.float64, device=dev)
    for _ in range(3):
        ssim_sum(a, b, acc, up, ws, kc=0.8 / a.numel(), tau=0.2, upstream=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        ssim_sum(a, b, acc, up, ws, kc=0.8 / a.numel(), tau=0.2, upstream=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    peak, kind = load_peaks()
    gbs = 72.0 * a.numel() / (ms / 1e3) / 1e9
    return {"kernel": "sgad_ssim (stats + grad, fused upstream)", "ms_per_view": ms,
            "achieved_gbs": gbs, "peak_gbs": peak, "frac": gbs / peak, "image": [h, w, c]}


def bench_render_init(dev, iters=3):
    """Render-based pose initialiser (tracker.py:354-426) at C4 size (room
    scene, 1200x680): wall time per IRLS-GN iteration (13 renders + halving
    candidates on the GPU, 6x6 solves on the host)."""
    import torch
    from paper_2603_21055_b200 import scenes
    from paper_2603_21055_b200.gaussians import PixelGaussianMap
    from paper_2603_21055_b200.geometry import Pose
    from paper_2603_21055_b200.tracker import init_pose_render
    intr, fa, fb, p, truth = scenes.config_render_init(intr_kw=scenes.C4_INTR,
                                                       scene=scenes.room_scene(0), device=dev)
    m = PixelGaussianMap(0, Pose.identity(), intr, p.base_depth, p.delta, p.color, p.log_radius,
                         p.opacity_logit, p.active_mask, dtype=torch.float64, device=dev)
    init_pose_render(fb, m, Pose.identity(), iters=1)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pose, ok = init_pose_render(fb, m, Pose.identity(), iters=iters)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    return {"metric": "render-based pose init (1200x680, IRLS-GN, central-difference "
                      "Jacobian through the GPU rasterizer)",
            "ms_per_iteration": dt / iters * 1e3, "iterations": iters, "ok": bool(ok)}


def bench_tracking(dev, which="c4size", iters=20, reps=5):
    """Secondary metric: GN iterations/s of the fused GICP normal equations
    (window fit of both frames, exact NN, host 6x6 solve), 20 GN iterations
    with convergence_eps = 0, timed with CUDA events around ``reps`` runs
    (the host solves are inside).  ``which``: "c4size" (1200x680 room scene,
    816 k correspondences) or "c2" (BASELINE config 1: 320x240, 76.8 k).
    Roofline: 84 B per correspondence for the linearisation (local centre +
    covariance 36 B, target centre + covariance + normal 48 B) plus 84 B for
    the candidate cost pass = 168 M bytes per GN iteration."""
    import numpy as np
    import torch
    from paper_2603_21055_b200 import tracker as T
    from paper_2603_21055_b200 import scenes
    from paper_2603_21055_b200.geometry import Intrinsics, Pose
    if which == "c2":
        intr, ref, qry, truth = scenes.config_c2(device=dev)
    else:
        intr = Intrinsics(**scenes.C4_INTR)
        prims = scenes.room_scene(0)
        ref = scenes.render_frame(prims, Pose.identity(), intr, 0, depth_noise_rel=0.01,
                                  device=dev)
        truth = scenes.se3_exp([0.01, -0.02, 0.015, 0.03, -0.01, 0.02])
        qry = scenes.render_frame(prims, truth, intr, 1, depth_noise_rel=0.01, device=dev)
    cfg = T.TrackerConfig(downsample_ratio=1, max_gicp_iters=iters, convergence_eps=0.0,
                          voxel_size=1e-4)
    g = T.GlobalGeomSet(cfg.voxel_size)
    ref_local = T.build_local_set(ref, cfg)
    torch.cuda.synchronize()
    t_ins = time.perf_counter()
    T.update_global_set(g, ref_local, Pose.identity())
    torch.cuda.synchronize()
    insert_ms = (time.perf_counter() - t_ins) * 1e3
    local = T.build_local_set(qry, cfg)
    T.gicp_align(local, g, Pose.identity(), cfg)  # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n_it = 0
    for _ in range(reps):
        pose, diag = T.gicp_align(local, g, Pose.identity(), cfg)
        n_it += diag.iterations + (0 if diag.iterations == iters else 1)
    e1.record()
    torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) / 1e3
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for _ in range(reps):
        T.build_local_set(qry, cfg)
    f1.record()
    torch.cuda.synchronize()
    fit_ms = f0.elapsed_time(f1) / reps
    # the next keyframe's insertion into the existing set (voxel gating +
    # grid rebuild over all members), as the tracking loop does per keyframe
    members = len(g)
    torch.cuda.synchronize()
    t_ins = time.perf_counter()
    added = T.update_global_set(g, local, pose)
    torch.cuda.synchronize()
    insert_next_ms = (time.perf_counter() - t_ins) * 1e3
    m = len(local)
    peak, peak_kind = load_peaks()
    it_s = dt / n_it
    achieved = 168.0 * m / it_s / 1e9
    return {"metric": f"tracking GN iterations/s ({which}: {intr.width}x{intr.height}, 5x5 window "
                      f"fit, exact NN, host solve)",
            "value": n_it / dt, "unit": "GN iters/s", "correspondences": m,
            "iterations_per_run": diag.iterations, "ms_per_iteration": it_s * 1e3,
            "fit_ms_per_frame": fit_ms, "global_insert_ms": insert_ms,
            "global_insert_next_ms": insert_next_ms, "global_insert_next_added": int(added),
            "global_members": members,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak,
                         "peak_source": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "bytes_per_iteration": 168 * m,
                         "note": "whole GN iteration (NN search + normal equations + cost pass "
                                 "+ 2 host round trips) against 168 B per correspondence"}}


def bench_tracking_rendered(dev, wc, key=3, iters=20, reps=3):
    """BASELINE config 4's tracking: a frame tracked (20 GN iterations)
    against geometry Gaussians fitted to the window's RENDERED depth, as the
    reference pipeline builds its global set (mapper.py:208-210,
    pipeline.py:346-349: D / A where the accumulated alpha A > 0.5).  The
    window maps (fp64 drop-in maps of the bench's window) render keyframe
    ``key``'s view with normalize_depth; the next keyframe's sensor depth is
    registered against it from keyframe ``key``'s pose."""
    import numpy as np
    import torch
    from paper_2603_21055_b200 import tracker as T
    from paper_2603_21055_b200.gaussians import PixelGaussianMap
    from paper_2603_21055_b200.geometry import pose_difference
    from paper_2603_21055_b200.rasterizer import splat
    from paper_2603_21055_b200.scenes import Frame
    maps = [PixelGaussianMap(i, wc.poses[i], wc.intr, p.base_depth, p.delta, p.color,
                             p.log_radius, p.opacity_logit, p.active_mask, dtype=torch.float64,
                             device=dev) for i, p in enumerate(wc.params)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = splat(maps, wc.poses[key], wc.intr, normalize_depth=True)
    geo = out.alpha > 0.5
    depth = torch.where(geo, out.depth, torch.zeros_like(out.depth)).float()
    cfg = T.TrackerConfig(downsample_ratio=1, max_gicp_iters=iters, convergence_eps=0.0,
                          voxel_size=1e-4)
    g = T.GlobalGeomSet(cfg.voxel_size)
    T.update_global_set(g, T.build_local_set(Frame(None, depth, geo, wc.intr, index=key), cfg),
                        wc.poses[key])
    torch.cuda.synchronize()
    build_ms = (time.perf_counter() - t0) * 1e3
    fr = wc.frames[key + 1]
    local = T.build_local_set(fr, cfg)
    T.gicp_align(local, g, wc.poses[key], cfg)  # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n_it = 0
    for _ in range(reps):
        pose, diag = T.gicp_align(local, g, wc.poses[key], cfg)
        n_it += max(diag.iterations, 1)
    e1.record()
    torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) / 1e3
    rot_err, t_err = pose_difference(pose, wc.poses[key + 1])
    return {"metric": "tracking GN iterations/s against rendered-geometry Gaussians "
                      f"(keyframe {key + 1} of the window vs keyframe {key}'s render, "
                      f"{wc.intr.width}x{wc.intr.height})",
            "value": n_it / dt, "unit": "GN iters/s", "correspondences": len(local),
            "global_members": len(g), "iterations_per_run": diag.iterations,
            "render_fit_insert_ms": build_ms, "pose_error_rad_m": [rot_err, t_err]}


def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(args):
    """``--gpus N`` without a torchrun environment: re-exec this command under
    torch.distributed.run with N ranks (one process per GPU, rendezvous on
    127.0.0.1), the launch the driver uses for N > 1."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    print(f"bench.py: launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)
    if args.launch_check:
        launch_check(args)
        return
    run_ours(args)


if __name__ == "__main__":
    main()
