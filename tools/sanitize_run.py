import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import stereo_synth as synth
import paper_1807_02044_b200 as fbs
for name in ("synthetic", "teddy", "kitti"):
    cfg = synth.CONFIGS[name]
    L, R = synth.frame(cfg, 1)
    m = fbs.FBS(cfg.W, cfg.H, cfg.d_min, cfg.d_max, cfg.radius, cfg.gamma_d, cfg.gamma_r)
    out = m.compute(torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda())
    torch.cuda.synchronize()
    print(name, float((out >= 0).float().mean()))
for rho in (0, 3, 6):
    cfg = synth.CONFIGS["synthetic"]
    L, R = synth.frame(cfg, 0)
    m = fbs.FBS(cfg.W, cfg.H, cfg.d_min, cfg.d_max, rho, cfg.gamma_d, cfg.gamma_r)
    out = m.compute(torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda()); torch.cuda.synchronize()
    print("rho", rho, float((out >= 0).float().mean()))
# the EMPTY-form instantiation on the textureless-heavy KITTI frame, and the
# debug-export instantiation
os.environ["FBS_EMPTY_FORM"] = "1"
cfg = synth.CONFIGS["kitti"]
L, R = synth.frame(cfg, 1)
m = fbs.FBS(cfg.W, cfg.H, cfg.d_min, cfg.d_max, cfg.radius, cfg.gamma_d, cfg.gamma_r)
out = m.compute(torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda()); torch.cuda.synchronize()
print("kitti empty-form", float((out >= 0).float().mean()))
del os.environ["FBS_EMPTY_FORM"]
cfg = synth.CONFIGS["synthetic"]
L, R = synth.frame(cfg, 0)
m = fbs.FBS(cfg.W, cfg.H, cfg.d_min, cfg.d_max, cfg.radius, cfg.gamma_d, cfg.gamma_r)
vols = m.volumes(torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda()); torch.cuda.synchronize()
print("export", [float(v.float().mean()) for v in vols])
