#!/usr/bin/env python
"""Top source lines by executed warp instructions (and stall samples) from an .ncu-rep.
usage: python scripts/ncu_inst_lines.py file.ncu-rep [topN]"""
import csv, subprocess, sys
rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
acc = {}
order = []
cur = None
for r in rows:
    if r and r[0] == "Line No" and len(r) > 5:
        hdr = r
        ii, si = hdr.index("Instructions Executed"), hdr.index("# Samples")
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0] != "":   # cuda source row aggregates its sass rows
        key = (r[0], r[1].strip()[:110])
        try:
            n, sm = int(r[ii]), int(r[si])
        except ValueError:
            continue
        a = acc.setdefault(key, [0, 0])
        a[0] += n; a[1] += sm
tot_i = sum(a[0] for a in acc.values()) or 1
tot_s = sum(a[1] for a in acc.values()) or 1
print(f"total warp instructions {tot_i}, samples {tot_s}")
for (ln, src), (n, sm) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*n/tot_i:5.1f}% inst {100*sm/tot_s:5.1f}% smp  L{ln:>5} {src}")
