import os, sys
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_2603_21055_b200.mapper import MapperConfig, WindowMapper
dev = torch.device("cuda", 0)
for name in ("c3", "c4"):
    wc = bench.make_config(name, dev)
    wm = WindowMapper(wc.frames, wc.poses, wc.intr, wc.params, MapperConfig(tau=0.0), device=dev)
    for v in (0, 3, 7):
        print(name, v, file=sys.stderr)
        wm.raster.prepare(wm._frames[v], wm.cam, want_coef=True)
