#!/usr/bin/env python
"""NEXT-1: runtime vs aggregation radius rho at the Teddy shape,
the shape of the paper's Fig. 7 (`fig.eva4`) including its rho = 6
operating point (344.16 Mde/s on a GTX 1080, P:L341 - context, not a target).
Runs bench.py once per radius on this GPU and prints one table (also written to
profiles/<tag>_radius_sweep.txt when a tag is given).

usage: python tools/sweep_radius.py [tag] [--steps K]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else None
    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 500
    rows = []
    for rho in range(0, 7):
        out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "teddy",
                              "--radius", str(rho), "--steps", str(steps), "--warmup", "10", "--no-extras"],
                             capture_output=True, text=True)
        d = json.loads(out.stdout.strip().splitlines()[-1])
        r = d["roofline"]
        rows.append((rho, (2 * rho + 1) ** 2, d["ms_per_step"], d["fps"], d["value"], r["frac"], r["achieved"]))
    lines = ["# Teddy-shaped 450x375, D=60, gamma_d=5, gamma_r=32, one B200; bench.py --no-extras",
             "# Mdisp/s = W*H*D*fps*1e-6 (Eq.(13) with the range width); paper (GTX 1080, rho=6): 344.16 Mde/s",
             f"{'rho':>3} {'K':>4} {'ms/frame':>9} {'fps':>8} {'Mdisp/s':>9} {'x paper':>8} {'agg TFLOP/s':>11} {'frac':>6}"]
    for rho, K, ms, fps, v, frac, ach in rows:
        lines.append(f"{rho:>3} {K:>4} {ms:>9.4f} {fps:>8.0f} {v:>9.0f} {v / 344.16:>8.0f} {ach:>11.2f} {frac:>6.3f}")
    txt = "\n".join(lines) + "\n"
    print(txt)
    if tag:
        open(os.path.join(ROOT, "profiles", f"{tag}_radius_sweep.txt"), "w").write(txt)


if __name__ == "__main__":
    main()
