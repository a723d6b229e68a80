#!/usr/bin/env python
"""Top source lines by warp-stall samples from an .ncu-rep (all files of the first kernel, or kernel index argv[3]).
usage: python scripts/ncu_hot_lines.py file.ncu-rep [topN] [kernel substring]"""
import csv, subprocess, sys, os
rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
want = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
blocks, cur, path = [], None, None
for r in rows:
    if r and r[0] == "File Path":
        path = r[1]
    elif r and r[0] == "Function Name":
        cur = {"name": r[1], "file": os.path.basename(path or "?"), "hdr": None, "lines": []}
        blocks.append(cur)
    elif r and r[0] == "Line No" and cur is not None and cur["hdr"] is None:
        cur["hdr"] = r
    elif cur is not None and cur["hdr"] is not None and r:
        cur["lines"].append(r)
names = []
for b in blocks:
    if b["name"] not in names:
        names.append(b["name"])
kname = next((n for n in names if want and want in n), names[0])
def num(x):
    try:
        return int(x)
    except ValueError:
        return 0
allsrc = []
for b in blocks:
    if b["name"] != kname:
        continue
    hdr = b["hdr"]
    si = hdr.index("# Samples")
    ii = hdr.index("Instructions Executed")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    for r in b["lines"]:
        if r[0] != "" and len(r) > si:
            allsrc.append((b["file"], r, si, ii, stall_cols, hdr))
tot = sum(num(r[si]) for _, r, si, _, _, _ in allsrc) or 1
toti = sum(num(r[ii]) for _, r, _, ii, _, _ in allsrc) or 1
print("==", kname[:100], "samples", tot, "warp-instructions", toti)
for f, r, si, ii, sc, hdr in sorted(allsrc, key=lambda x: -num(x[1][x[2]]))[:top]:
    st = sorted(((num(r[i]), hdr[i]) for i in sc), reverse=True)[:3]
    print(f"{num(r[si])/tot:6.1%} i{num(r[ii])/toti:5.1%} {f[:12]:12s} L{r[0]:>4} {r[1].strip()[:70]:70s} {' '.join(f'{n[6:]}:{c}' for c, n in st if c)}")
