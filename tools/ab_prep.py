"""A/B timing of the preparation (K1-K3, one C4 view, isolated, CUDA events,
median of 20) for alternative libsgad builds:
python tools/ab_prep.py [c3|c4] variants/a.so variants/b.so ..."""
import os
import subprocess
import sys

CODE = r'''
import os, sys, statistics
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_2603_21055_b200.mapper import MapperConfig, WindowMapper
dev = torch.device("cuda", 0)
wc = bench.make_config(sys.argv[1], dev)
wm = WindowMapper(wc.frames, wc.poses, wc.intr, wc.params, MapperConfig(tau=0.0), device=dev)
r = wm.raster
ns, npairs = r.prepare(wm._frames[3], wm.cam, want_coef=True)
ts = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    r.prepare_async(wm._frames[3], wm.cam, want_coef=True)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"{statistics.median(ts):.3f} ms (min {min(ts):.3f})  survivors {ns} pairs {npairs}")
'''
cfg = sys.argv[1]
for lib in sys.argv[2:]:
    env = dict(os.environ, SGAD_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", CODE, cfg], capture_output=True, text=True, env=env)
    print(f"{lib:34s} {out.stdout.strip() or out.stderr[-300:]}", flush=True)
