"""K5 contribution coincidence count (diagnostic build -DSGAD_K5_COUNT): one
eager C4 window step; per view, contributions vs distinct (entry, warp
iteration) pairs -- the most a warp-level pre-reduction could merge."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2603_21055_b200.mapper import MapperConfig, WindowMapper
dev = torch.device("cuda", 0)
wc = bench.make_config(sys.argv[1] if len(sys.argv) > 1 else "c4", dev)
wm = WindowMapper(wc.frames, wc.poses, wc.intr, wc.params, MapperConfig(tau=0.0), device=dev)
wm.use_graph = False
wm.step(sync_loss=True)
