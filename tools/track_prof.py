"""Host-side profile of gicp_align at c4size (cProfile, top functions by own time)
and the split of a GN iteration into GPU-busy and host time."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_21055_b200 import tracker as T
from paper_2603_21055_b200 import scenes
from paper_2603_21055_b200.geometry import Intrinsics, Pose

dev = torch.device("cuda", 0)
intr = Intrinsics(**scenes.C4_INTR)
prims = scenes.room_scene(0)
ref = scenes.render_frame(prims, Pose.identity(), intr, 0, depth_noise_rel=0.01, device=dev)
truth = scenes.se3_exp([0.01, -0.02, 0.015, 0.03, -0.01, 0.02])
qry = scenes.render_frame(prims, truth, intr, 1, depth_noise_rel=0.01, device=dev)
cfg = T.TrackerConfig(downsample_ratio=1, max_gicp_iters=20, convergence_eps=0.0, voxel_size=1e-4)
g = T.GlobalGeomSet(cfg.voxel_size)
T.update_global_set(g, T.build_local_set(ref, cfg), Pose.identity())
local = T.build_local_set(qry, cfg)
T.gicp_align(local, g, Pose.identity(), cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    T.gicp_align(local, g, Pose.identity(), cfg)
torch.cuda.synchronize()
print("wall ms per GN iteration", (time.perf_counter() - t0) / 100 * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    T.gicp_align(local, g, Pose.identity(), cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
