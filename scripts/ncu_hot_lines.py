#!/usr/bin/env python
"""Top source lines by warp-stall samples from an .ncu-rep (per kernel launch id).
usage: python scripts/ncu_hot_lines.py file.ncu-rep [topN]"""
import csv, subprocess, sys
rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
# split per kernel: a block starts with "File Path" / "Function Name"
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Function Name":
        cur = {"name": r[1], "hdr": None, "lines": []}
        blocks.append(cur)
    elif r and r[0] == "Line No" and cur is not None and cur["hdr"] is None:
        cur["hdr"] = r
    elif cur is not None and cur["hdr"] is not None and r and r[0] not in ("File Path",):
        cur["lines"].append(r)
for b in blocks[:1] if len(sys.argv) <= 3 else blocks:
    hdr = b["hdr"]
    si = hdr.index("# Samples")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    def num(x):
        try:
            return int(x)
        except ValueError:
            return 0
    src = [r for r in b["lines"] if r[0] != "" and len(r) > si]   # cuda source rows
    tot = sum(num(r[si]) for r in src) or 1
    print("==", b["name"][:90], "samples", tot)
    for r in sorted(src, key=lambda r: -num(r[si]))[:top]:
        st = sorted(((num(r[i]), hdr[i]) for i in stall_cols), reverse=True)[:3]
        print(f"{num(r[si])/tot:6.1%} L{r[0]:>4} {r[1].strip()[:80]:80s} {' '.join(f'{n}:{c}' for c, n in st if c)}")
