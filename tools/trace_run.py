"""Timeline of CTA 0 of the warp-specialised walker (trace builds: -DFBS_TRACE,
tools/build_variants.py trace='-DFBS_TRACE'), one Teddy frame.  Prints per-phase
producer and per-chunk consumer durations in SM cycles.
  FBS_LIB=paper_1807_02044_b200/libfbs_exp_trace.so python tools/trace_run.py [config]"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import stereo_synth as synth  # noqa: E402
import torch  # noqa: E402
import paper_1807_02044_b200 as fbs  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "teddy"]
lib = fbs.load_library()
lib.fbs_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
L, R = (torch.from_numpy(x).cuda() for x in synth.frame(cfg, 0))
m = fbs.FBS(cfg.W, cfg.H, cfg.d_min, cfg.d_max, cfg.radius, cfg.gamma_d, cfg.gamma_r)
for _ in range(3):
    m.compute(L, R)
torch.cuda.synchronize()
buf = np.zeros(8192, dtype=np.uint64)
assert lib.fbs_debug_trace(m.h, buf.ctypes.data, 8192) == 0
prod = buf[:4000].reshape(-1, 4).astype(np.int64)
prod = prod[prod[:, 0] != 0]
chunkflag = (buf[:4000].reshape(-1, 4)[: len(prod), 3] >> np.uint64(63)).astype(bool)
prod[:, 3] &= (1 << 62) - 1
cons = buf[4096:8096].reshape(-1, 4).astype(np.int64)
cons = cons[cons[:, 0] != 0]
t0 = min(prod[0, 0], cons[0, 0])
print(f"producer phases: {len(prod)} (chunks {chunkflag.sum()}), span {prod[-1, 3] - t0} cycles")
d = np.diff(prod, axis=1)
print("  mean cycles: empty-wait %.0f  issue+tma-wait %.0f  compute %.0f   (per phase, total %.0f)" %
      (d[:, 0].mean(), d[:, 1].mean(), d[:, 2].mean(), (prod[:, 3] - prod[:, 0]).mean()))
gaps = prod[1:, 0] - prod[:-1, 3]
print("  gap between phases %.0f" % gaps.mean())
print(f"consumer chunks: {len(cons)}, span {cons[-1, 3] - t0}")
d = np.diff(cons, axis=1)
print("  mean cycles: full-wait %.0f  stream+emit %.0f  wta+record %.0f   (per chunk, total %.0f)" %
      (d[:, 0].mean(), d[:, 1].mean(), d[:, 2].mean(), (cons[:, 3] - cons[:, 0]).mean()))
for i in range(min(12, len(prod))):
    print("  P", i, "chunk" if chunkflag[i] else "fill ", (prod[i] - t0).tolist())
for i in range(min(12, len(cons))):
    print("  C", i, (cons[i] - t0).tolist())
