"""bench.py's C2 tracking metric alone (320x240, 76.8 k correspondences)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
print(json.dumps(bench.bench_tracking(torch.device("cuda", 0), "c2")))
