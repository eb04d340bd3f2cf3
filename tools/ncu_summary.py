#!/usr/bin/env python
"""Summarise an ncu --set full report: SOL, issue, stalls, pipes, DRAM bytes,
and (optionally) SASS opcode mix with stall samples.  Usage:
  python tools/ncu_summary.py report.ncu-rep [--sass]"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum", "local_load", "sm__cycles_elapsed.avg.per_second",
        "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
        "sm__cycles_active.avg", "gpc__cycles_elapsed.max"]


def ncu(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    rows = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    hdr, units = rows[0], rows[1]
    for row in rows[2:]:
        name = row[hdr.index("Kernel Name")]
        print("==", name[:80])
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k} = {row[i]} {units[i]}")
        st = []
        for i, k in enumerate(hdr):
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    v = float(row[i])
                except ValueError:
                    continue
                if v >= 0.05:
                    st.append((v, k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        print("  stalls/issue:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)))
    if "--sass" in sys.argv:
        rows = list(csv.reader(io.StringIO(ncu([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
        hdr = rows[1]
        ia, ie = hdr.index("Source"), hdr.index("Instructions Executed")
        iss = hdr.index("Warp Stall Sampling (All Samples)")
        ops, st = collections.Counter(), collections.Counter()
        for r in rows[2:]:
            if len(r) <= ie:
                continue
            try:
                n = int(r[ie].replace(",", "")); s = int(r[iss].replace(",", ""))
            except ValueError:
                continue
            toks = r[ia].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") else toks[0]
            ops[op.split(".")[0]] += n
            st[op.split(".")[0]] += s
        tot, tots = sum(ops.values()), sum(st.values())
        print(f"  SASS executed {tot}, stall samples {tots}")
        for op, n in ops.most_common(18):
            print(f"    {op:8s} {100 * n / tot:5.1f}% of instr, {100 * st[op] / max(1, tots):5.1f}% of stall samples")


if __name__ == "__main__":
    main()
