"""Tracking micro-benchmark at 1200x680 (bench.py's secondary metric)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
print(json.dumps(bench.bench_tracking(torch.device("cuda", 0), iters=int(sys.argv[1]) if len(sys.argv) > 1 else 20,
                                      reps=int(sys.argv[2]) if len(sys.argv) > 2 else 5)))
