#!/usr/bin/env python
"""Warp-stall reason totals (sampling) for one kernel of an .ncu-rep.  usage: ncu_stalls.py file.ncu-rep [kernel substring]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, hdr, tot, name = None, None, collections.Counter(), None
for r in rows:
    if r and r[0] == "Kernel Name":
        name = r[1]; hdr = None
    elif r and r[0] == "Address":
        hdr = r
    elif hdr and r and (want is None or want in (name or "")):
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h and i < len(r):
                try: tot[h] += int(r[i])
                except ValueError: pass
        tot["#instr_rows"] += 1
s = sum(v for k, v in tot.items() if k.startswith("stall_")) or 1
print("sass rows", tot["#instr_rows"])
for k, v in tot.most_common():
    if k.startswith("stall_"): print(f"{k:28s} {v:8d} {v/s:6.1%}")
