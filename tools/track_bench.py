"""Tracking micro-benchmark at 1200x680 (bench.py's secondary metric)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
if os.environ.get("GICP_HOST") == "1":
    from paper_2603_21055_b200 import tracker
    tracker.GICP_DEVICE_LOOP = False
print(json.dumps(bench.bench_tracking(torch.device("cuda", 0), iters=int(sys.argv[1]) if len(sys.argv) > 1 else 20,
                                      reps=int(sys.argv[2]) if len(sys.argv) > 2 else 5)))
