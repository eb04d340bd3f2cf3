#!/usr/bin/env python
"""NEXT-1: runtime vs aggregation radius rho at the Teddy shape,
the shape of the paper's Fig. 7 (`fig.eva4`) including its rho = 6
operating point (344.16 Mde/s on a GTX 1080, P:L341 - context, not a target).
Runs bench.py once per radius on this GPU and prints one table (also written to
profiles/<tag>_radius_sweep.txt when a tag is given).

usage: python tools/sweep_radius.py [tag] [--steps K] [--path volume|fused]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else None
    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 500
    path = sys.argv[sys.argv.index("--path") + 1] if "--path" in sys.argv else "volume"
    rows = []
    for rho in range(0, 11 if path == "volume" else 7):
        out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "teddy", "--path", path,
                              "--radius", str(rho), "--steps", str(steps), "--warmup", "10", "--no-extras"],
                             capture_output=True, text=True)
        d = json.loads(out.stdout.strip().splitlines()[-1])
        r = d["roofline"]
        rows.append((rho, (2 * rho + 1) ** 2, d["ms_per_step"], d["fps"], d["value"], r["frac"], r["achieved"]))
    lines = [f"# Teddy-shaped 450x375, D=60, gamma_d=5, gamma_r=32, one B200; bench.py --no-extras --path {path}",
             "# Mdisp/s = W*H*D*fps*1e-6 (Eq.(13) with the range width); paper (GTX 1080, rho=6): 344.16 Mde/s",
             f"{'rho':>3} {'K':>4} {'ms/frame':>9} {'fps':>8} {'Mdisp/s':>9} {'x paper':>8} {'agg TFLOP/s':>11} {'frac':>6}"]
    for rho, K, ms, fps, v, frac, ach in rows:
        lines.append(f"{rho:>3} {K:>4} {ms:>9.4f} {fps:>8.0f} {v:>9.0f} {v / 344.16:>8.0f} {ach:>11.2f} {frac:>6.3f}")
    t = {r[0]: r[2] for r in rows}
    if 7 in t and 5 in t and 6 in t:  # the paper's Fig. 7 remark (reading R#25)
        lines.append(f"# runtime ratio rho=7 / rho=5 = {t[7] / t[5]:.2f}, rho=7 / rho=6 = {t[7] / t[6]:.2f} "
                     "(paper, P:L345: 'the processing speed is doubled' when rho goes from 5-6 to 7; "
                     "read as runtime doubling, R#25)")
    txt = "\n".join(lines) + "\n"
    print(txt)
    if tag:
        open(os.path.join(ROOT, "profiles", f"{tag}_radius_sweep_{path}.txt"), "w").write(txt)


if __name__ == "__main__":
    main()
