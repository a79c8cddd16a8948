"""Prepare (K1-K3) one view of a window configuration, inside a CUDA
profiler range after warm-up: python tools/prep_once.py [c3|c4|c5] [view]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2603_21055_b200.mapper import MapperConfig, WindowMapper

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
view = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda", 0)
wc = bench.make_config(name, dev)
wm = WindowMapper(wc.frames, wc.poses, wc.intr, wc.params, MapperConfig(tau=0.0), device=dev)
r = wm.raster
for _ in range(2):
    ns, npairs = r.prepare(wm._frames[view], wm.cam, want_coef=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.profiler.start()
e0.record()
r.prepare_async(wm._frames[view], wm.cam, want_coef=True)
e1.record()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"prepare (async, isolated) {e0.elapsed_time(e1):.3f} ms; survivors {ns} pairs {npairs}")
