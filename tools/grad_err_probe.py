import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from helpers import forced_params, rel_err
from paper_2603_21055_b200 import scenes
from paper_2603_21055_b200.mapper import MapperConfig, WindowMapper
g = dict(np.load("tests/golden/bench_c3_forced.npz"))
wc = scenes.config_c3(); params = forced_params(wc.params); v = int(g["view"])
wm = WindowMapper(wc.frames, wc.poses, wc.intr, params, MapperConfig(tau=0.0))
for rep in range(4):
    wm.grad.zero_(); wm.loss_acc.zero_(); wm.render_view_grads(v)
    gr = wm.grad.view(wm.F, wm.HW, 8)[..., :6].permute(0, 2, 1).double().cpu().numpy()
    got = gr.transpose(0, 2, 1).reshape(-1, 6)[g["gs"]]
    errs = [rel_err(got[:, c], g["g_sample"][:, c], floor_frac=1e-3) for c in range(6)]
    c = 2; want = g["g_sample"][:, c]; sc = np.abs(want).max(); den = np.maximum(np.abs(want), 1e-3*sc)
    i = np.argmax(np.abs(got[:, c]-want)/den)
    print(os.environ.get("SGAD_LIB","default")[-12:], ["%.2e" % e for e in errs], "worst logit: got %.4e want %.4e max %.4e" % (got[i,c], want[i], sc), flush=True)
