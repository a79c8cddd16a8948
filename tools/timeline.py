"""Per-view event timeline of one C4 window step (prepare on the side stream,
compositing on the main stream): python tools/timeline.py [c4]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2603_21055_b200.mapper import MapperConfig, WindowMapper
dev = torch.device("cuda", 0)
wc = bench.make_config(sys.argv[1] if len(sys.argv) > 1 else "c4", dev)
wm = WindowMapper(wc.frames, wc.poses, wc.intr, wc.params, MapperConfig(tau=0.0), device=dev)
for _ in range(3):
    wm.step()
torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
timing = []
t0.record()
wm.step(timing=timing)
t1.record()
torch.cuda.synchronize()
print(f"step {t0.elapsed_time(t1):.2f} ms")
for kind, a, b, v, ns, npairs in timing:
    print(f"{kind:5s} view {v}  start {t0.elapsed_time(a):7.2f}  end {t0.elapsed_time(b):7.2f}  dur {a.elapsed_time(b):6.2f}")
