"""Build libfbs.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = [os.path.join(HERE, "csrc", "fbs_capi.cu")]
DEPS = SRC + [os.path.join(HERE, "csrc", "fbs_kernels.cuh"), os.path.join(HERE, "csrc", "fbs_fused.cuh"), os.path.join(HERE, "csrc", "fbs_ws.cuh"), os.path.join(HERE, "csrc", "fbs_volume.cuh"), os.path.join(ROOT, "include", "fbs.h")]
OUT = os.path.join(HERE, "libfbs.so")

# Whole-module device compilation: `--split-compile` partitions the module and changes
# the code NVVM generates for every kernel (k_agg<4>: 7,248 instructions split vs 7,000
# whole; A/B on one B200: Teddy 6,610 -> 6,742 frames/s, KITTI +2.2 %, Tsukuba +2.7 %),
# at ~4 min instead of ~1.5 min of build time.  FBS_SPLIT_COMPILE=1 restores the split
# build for quick experiment builds.
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"] + (
                  ["--split-compile=0"] if os.environ.get("FBS_SPLIT_COMPILE") == "1" else [])


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(OUT) and all(os.path.getmtime(OUT) >= os.path.getmtime(d) for d in DEPS):
        return OUT
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    tmp = OUT + f".tmp{os.getpid()}"
    cmd = [nvcc, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", tmp, *SRC]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libfbs.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, OUT)
    with open(os.path.join(HERE, "csrc", "ptxas_info.txt"), "w") as f:
        f.write(res.stderr)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
