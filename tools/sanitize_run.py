"""Workload for compute-sanitizer (memcheck / racecheck / synccheck) over every
kernel path of libfbs.so: both implementation paths on synthetic, Teddy and a
textureless-heavy KITTI frame, radii 0/3/6 (+ 8, 10 on the volume path), the
debug-export instantiations, band handles, a batch (the fused path's multi-frame
launch), the disparity-range split (KEYS) and the sparse search range (RANGED).
  compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import stereo_synth as synth  # noqa: E402
import paper_1807_02044_b200 as fbs  # noqa: E402
from paper_1807_02044_b200 import dist as fdist  # noqa: E402


def dev(cfg, i):
    L, R = synth.frame(cfg, i)
    return torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda()


for path in ("volume", "fused"):
    for name in ("synthetic", "teddy", "kitti"):
        cfg = synth.CONFIGS[name]
        L, R = dev(cfg, 1)
        m = fbs.FBS(cfg.W, cfg.H, cfg.d_min, cfg.d_max, cfg.radius, cfg.gamma_d, cfg.gamma_r, path=path)
        out = m.compute(L, R)
        torch.cuda.synchronize()
        print(path, name, float((out >= 0).float().mean()))
    cfg = synth.CONFIGS["synthetic"]
    L, R = dev(cfg, 0)
    for rho in ((0, 3, 6, 8, 10) if path == "volume" else (0, 3, 6)):
        m = fbs.FBS(cfg.W, cfg.H, cfg.d_min, cfg.d_max, rho, cfg.gamma_d, cfg.gamma_r, path=path)
        out = m.compute(L, R)
        torch.cuda.synchronize()
        print(path, "rho", rho, float((out >= 0).float().mean()))
    m = fbs.FBS(cfg.W, cfg.H, cfg.d_min, cfg.d_max, cfg.radius, cfg.gamma_d, cfg.gamma_r, path=path)
    vols = m.volumes(L, R)
    torch.cuda.synchronize()
    print(path, "export", [float(v.float().mean()) for v in vols])
    cfg = synth.CONFIGS["tsukuba"]
    Ls, Rs = zip(*(dev(cfg, i) for i in range(3)))
    m = fbs.FBS(cfg.W, cfg.H, cfg.d_min, cfg.d_max, cfg.radius, cfg.gamma_d, cfg.gamma_r, path=path)
    outb = m.compute_batch(torch.stack(Ls), torch.stack(Rs))
    mb = fbs.FBS(cfg.W, cfg.H, cfg.d_min, cfg.d_max, cfg.radius, cfg.gamma_d, cfg.gamma_r, path=path, rows=(100, 180))
    band = mb.compute_rows(Ls[0], Rs[0], 100, 180)
    torch.cuda.synchronize()
    print(path, "batch + band", float((outb >= 0).float().mean()), float((band >= 0).float().mean()))

cfg = synth.CONFIGS["kitti"]
L, R = dev(cfg, 0)
keys_l, keys_r, recs = [], [], []
for lo, hi in fdist.drange_split(cfg.d_min, cfg.d_max, 3):
    a, b = fdist.handle_range(cfg.d_min, cfg.d_max, lo, hi)
    kl, kr, rec = fbs.FBS(cfg.W, cfg.H, a, b, cfg.radius, cfg.gamma_d, cfg.gamma_r).compute_keys(L, R, lo, hi)
    keys_l.append(kl); keys_r.append(kr); recs.append(rec)
kl, rec = fdist.reduce_keys_local(keys_l, recs)
kr, _ = fdist.reduce_keys_local(keys_r, recs)
out = fbs.finalize_keys(cfg.W, cfg.H, cfg.d_min, cfg.d_max, kl, kr, rec.contiguous())
m = fbs.FBS(cfg.W, cfg.H, cfg.d_min, cfg.d_max, cfg.radius, cfg.gamma_d, cfg.gamma_r)
seed = m.compute(L, R)
rl, rr = m.suggest_ranges(seed, 3)
outr = m.compute_ranged(L, R, rl, rr)
torch.cuda.synchronize()
print("drange split", float((out >= 0).float().mean()), "sparse range", float((outr >= 0).float().mean()))
