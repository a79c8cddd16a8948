"""One C4 window iteration inside a CUDA profiler range (for ncu
--profile-from-start off): python tools/step_once.py [c3|c4|c5] [warmup]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2603_21055_b200.mapper import MapperConfig, WindowMapper

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda", 0)
wc = bench.make_config(name, dev)
wm = WindowMapper(wc.frames, wc.poses, wc.intr, wc.params, MapperConfig(tau=0.0), device=dev)
for _ in range(warm):
    wm.step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
wm.step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("step ok", wm.counts())
