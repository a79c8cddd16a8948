"""Wall-time profile of GlobalGeomSet insertion at c4size (816 k members)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_21055_b200 import tracker as T
from paper_2603_21055_b200 import scenes
from paper_2603_21055_b200.geometry import Intrinsics, Pose

dev = torch.device("cuda", 0)
intr = Intrinsics(**scenes.C4_INTR)
ref = scenes.render_frame(scenes.room_scene(0), Pose.identity(), intr, 0, depth_noise_rel=0.01,
                          device=dev)
cfg = T.TrackerConfig(downsample_ratio=1, voxel_size=1e-4)
loc = T.build_local_set(ref, cfg)
for _ in range(2):
    g = T.GlobalGeomSet(cfg.voxel_size)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    T.update_global_set(g, loc, Pose.identity())
    torch.cuda.synchronize()
    print("insert ms", (time.perf_counter() - t0) * 1e3)
g = T.GlobalGeomSet(cfg.voxel_size)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
T.update_global_set(g, loc, Pose.identity())
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
