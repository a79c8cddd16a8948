import sys, time, torch, numpy as np
sys.path.insert(0, '.')
from paper_2603_21055_b200 import scenes
from paper_2603_21055_b200.gaussians import PixelGaussianMap
from paper_2603_21055_b200.geometry import Pose, se3_exp
from paper_2603_21055_b200.tracker import _RenderResiduals
dev = torch.device("cuda", 0)
intr, fa, fb, p, truth = scenes.config_render_init(intr_kw=scenes.C4_INTR, scene=scenes.room_scene(0), device=dev)
m = PixelGaussianMap(0, Pose.identity(), intr, p.base_depth, p.delta, p.color, p.log_radius, p.opacity_logit, p.active_mask, dtype=torch.float64, device=dev)
res = _RenderResiduals(fb, m, 4.0)
poses = [se3_exp(np.eye(6)[k % 6] * 1e-4 * (1 if k % 2 == 0 else -1)) for k in range(12)]
rows = torch.empty((12, res.n), dtype=torch.float64, device=dev)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res.batch(poses, rows); torch.cuda.synchronize(); t1 = time.perf_counter()
    for i, q in enumerate(poses): res(q, out=rows[i])
    torch.cuda.synchronize(); t2 = time.perf_counter()
    from paper_2603_21055_b200.rasterizer import build_frames
    for q in poses: build_frames([m], q, set())
    t3 = time.perf_counter()
    print(f"batch {1e3*(t1-t0):.1f} ms  sequential {1e3*(t2-t1):.1f} ms  build_frames x12 {1e3*(t3-t2):.1f} ms")
r = rows[0].clone(); jac = ((rows[0::2] - rows[1::2]) / 2e-4).T
torch.cuda.synchronize(); t0 = time.perf_counter()
xi = np.zeros(6)
for _ in range(3):
    r_pred = r + jac @ torch.as_tensor(xi, device=dev)
    wts = 1.0 / torch.clamp(r_pred.abs(), min=1e-3)
    hw = (jac.T @ (jac * wts[:, None])).cpu().numpy(); gw = (jac.T @ (wts * r)).cpu().numpy()
    xi = np.linalg.lstsq(hw, -gw, rcond=None)[0]
torch.cuda.synchronize(); print(f"irls {1e3*(time.perf_counter()-t0):.1f} ms")
