#!/usr/bin/env python
"""Per-code-region stall breakdown of an ncu source page (SASS): consecutive
instructions with the same execution count form a region."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 12
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[1]
ia, ie, iad = h.index("Source"), h.index("Instructions Executed"), h.index("Address")
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
ir = [h.index(k) for k in reasons]
groups = []
for r in rows[2:]:
    if len(r) <= ie:
        continue
    try:
        n = int(r[ie].replace(",", ""))
        st = [int(r[i].replace(",", "")) for i in ir]
    except ValueError:
        continue
    toks = r[ia].split()
    op = (toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")).split(".")[0]
    if groups and groups[-1]["n"] == n:
        g = groups[-1]
    else:
        g = dict(start=r[iad], n=n, lines=0, st=[0] * len(ir), ops=collections.Counter())
        groups.append(g)
    g["lines"] += 1
    g["ops"][op] += 1
    g["st"] = [a + b for a, b in zip(g["st"], st)]
tot = sum(sum(g["st"]) for g in groups)
for g in sorted(groups, key=lambda g: -sum(g["st"]))[:topn]:
    s = sum(g["st"])
    top = sorted(zip(g["st"], reasons), reverse=True)[:5]
    print(f"{g['start']} exec={g['n']:7d} lines={g['lines']:5d} stall={100 * s / tot:5.1f}%  ops={dict(g['ops'].most_common(3))}")
    print("      " + ", ".join(f"{n[6:]}={100 * v / max(1, s):.0f}%" for v, n in top))
