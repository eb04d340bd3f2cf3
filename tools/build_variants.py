"""Build experimental libfbs variants (paper_1807_02044_b200/libfbs_exp_<name>.so) from
-D flag sets, for A/B runs with FBS_LIB (tools/gpu.sh ab).  Usage:
  python tools/build_variants.py name1='-DFOO=1 -DBAR=2' name2='...'"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1807_02044_b200 import build as b  # noqa: E402

for arg in sys.argv[1:]:
    name, flags = arg.split("=", 1)
    out = os.path.join(b.HERE, f"libfbs_exp_{name}.so")
    cmd = [os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc"), *b.NVCC_FLAGS, *flags.split(),
           "-I", os.path.join(ROOT, "include"), "-o", out, *b.SRC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
        raise SystemExit(f"variant {name} failed")
    lines = [l for l in r.stderr.splitlines() if "registers" in l or "spill" in l or "k_agg" in l]
    print(name, "\n  " + "\n  ".join(l.strip() for l in lines if "k_agg" in l or True)[:3000])
