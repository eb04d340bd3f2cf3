"""One small frame through the C ABI (for compute-sanitizer runs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import stereo_synth as synth
import paper_1807_02044_b200 as fbs
W, H, dmin, dmax, rho = (int(v) for v in (sys.argv[1:6] if len(sys.argv) > 5 else (64, 48, 0, 15, 3)))
L, R, _, _ = synth.layered(W, H, dmin, dmax, 7, p_flat=0.3)
m = fbs.FBS(W, H, dmin, dmax, rho, 5.0, 32.0)
out = m.compute(torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda())
torch.cuda.synchronize()
print("ok", float((out >= 0).float().mean()))
