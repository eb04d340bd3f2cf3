#!/usr/bin/env python
"""Turn the ncu captures of a GPU session (gpurun_out/) into the committed
summaries under profiles/ (round-tagged):

  profiles/<tag>_launches_teddy.txt   per-kernel share of the step from the
                                      `ncu --metrics gpu__time_duration.sum` launch list
  profiles/<tag>_<kernel>_ncu.txt     SOL / issue / stall / DRAM summary + code regions
  profiles/ncu_summary.json           per-launch DRAM bytes of the aggregation kernel
                                      (bench.py's roofline "traffic")

usage: python tools/make_profiles.py <tag> [gpurun_out/<tag>] [--out DIR]
(--out: write the summaries elsewhere, e.g. on the GPU box into gpurun_out/, whose
.ncu-rep files are too large to bring back)
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(cmd):
    return subprocess.run(cmd, capture_output=True, text=True).stdout


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    per = collections.defaultdict(list)
    for r in rows[hdr_i + 1:]:
        if len(r) > iv and r[im] == "gpu__time_duration.sum":
            per[r[ik].split("(")[0]].append(float(r[iv].replace(",", "")))
    return per


KERNELS = {"volume": ("k_cost", "k_agg", "k_finalize"), "fused": ("k_prep", "k_fbs", "k_final")}
CAPTURES = (("agg", "prof_agg_teddy", "volume"), ("cost", "prof_cost_teddy", "volume"),
            ("fbsws", "prof_fbsws_teddy", "fused"))


def main():
    args = [a for a in sys.argv[1:]]
    out = os.path.join(ROOT, "profiles")
    if "--out" in args:
        i = args.index("--out")
        out = args[i + 1]
        del args[i:i + 2]
    tag = args[0]
    src = args[1] if len(args) > 1 else os.path.join(ROOT, "gpurun_out", tag)
    os.makedirs(out, exist_ok=True)
    sp = os.path.join(out, "ncu_summary.json")
    summary = json.load(open(sp)) if os.path.exists(sp) else {}
    summary = {k: v for k, v in summary.items() if "/" in k or k == "note"}  # drop the r01 layout
    for path, names in KERNELS.items():
        lp = os.path.join(src, f"launches_teddy_{path}.csv")
        if not os.path.exists(lp):
            continue
        per = launches(lp)
        ours = {k: v for k, v in per.items() if any(n in k for n in names)}
        tot = sum(sum(v) for v in ours.values())
        lines = [f"# {tag}: ncu launch list, Teddy 450x375 D=60 rho=4, {path} path "
                 "(bench.py --path {path} --steps 20 --warmup 3 --no-extras --no-graph)".replace("{path}", path),
                 "# gpu__time_duration.sum, --clock-control none; cold-cache, serialised: compare SHARES", ""]
        for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"{k:50s} launches={len(v):4d} mean={sum(v) / len(v) / 1e3:9.2f} us "
                         f"share={100 * sum(v) / tot:5.1f}%")
        open(os.path.join(out, f"{tag}_launches_teddy_{path}.txt"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))
    for name, rep, path in CAPTURES:
        rp = os.path.join(src, rep + ".ncu-rep")
        if not os.path.exists(rp):
            continue
        s = run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rp, "--sass"])
        r = run([sys.executable, os.path.join(ROOT, "tools", "ncu_regions.py"), rp, "12"])
        open(os.path.join(out, f"{tag}_{name}_teddy_ncu.txt"), "w").write(
            f"# {tag}: ncu --set full --clock-control none --import-source on, Teddy config, {path} path, "
            "one launch (both sides)\n" + s + "\n# code regions by stall samples (tools/ncu_regions.py)\n" + r)
        raw = list(csv.reader(io.StringIO(run(["ncu", "-i", rp, "--page", "raw", "--csv"]))))
        h, v = raw[0], raw[2]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(v[h.index("dram__bytes_read.sum")]) * scale[raw[1][h.index("dram__bytes_read.sum")]]
        wr = float(v[h.index("dram__bytes_write.sum")]) * scale[raw[1][h.index("dram__bytes_write.sum")]]
        key = f"teddy/{path}"
        if name in ("agg", "fbsws"):  # the dominant kernel of the path: bench.py's roofline traffic
            summary.setdefault(key, {})["dram_bytes_per_launch"] = rd + wr
            summary[key]["kernel"] = v[h.index("Kernel Name")][:40]
        summary.setdefault(key, {})[f"{name}_dram_read_bytes"] = rd
        summary[key][f"{name}_dram_write_bytes"] = wr
        summary[key][f"{name}_duration_us"] = float(v[h.index("gpu__time_duration.sum")])
    summary["note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch of the path's dominant kernel "
                       "from one ncu --set full capture (replays flush caches: cold-L2 upper bound)")
    json.dump(summary, open(sp, "w"), indent=1)
    for f in sorted(os.listdir(src)):
        if f.startswith("bench_") and f.endswith(".json"):
            txt = open(os.path.join(src, f)).read().strip()
            if txt:
                open(os.path.join(out, f"{tag}_{f}"), "w").write(txt + "\n")


if __name__ == "__main__":
    main()
