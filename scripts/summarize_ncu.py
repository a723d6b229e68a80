#!/usr/bin/env python
"""Summarise ncu outputs brought back in gpurun_out/ into small tracked files under profiles/.

  python scripts/summarize_ncu.py launches gpurun_out/launches.csv profiles/r01_launches.md [skip]
  python scripts/summarize_ncu.py full gpurun_out/prof_x.ncu-rep profiles/r01_x_full.md
"""
import csv
import re
import subprocess
import sys
from collections import OrderedDict

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "smsp__inst_executed.sum", "lts__t_bytes.sum", "dram__cycles_active.avg",
]


def short(name):
    name = re.sub(r"\(.*", "", name)
    return name.replace("void ", "").replace("dg::", "")


def launches(src, dst, skip=0):
    rows = [r for r in csv.reader(l for l in open(src) if l.startswith('"'))]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    acc = OrderedDict()
    total = 0.0
    for r in rows[1 + skip:]:
        v = float(r[vi].replace(",", ""))
        us = v / 1000.0 if r[ui] in ("ns", "nsecond") else (v if r[ui] in ("us", "usecond") else v * 1000.0)
        k = short(r[ki])
        a = acc.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += us
        total += us
    with open(dst, "w") as f:
        f.write(f"# ncu launch list summary ({src}; {len(rows) - 1 - skip} launches, cold-cache serialised times)\n\n")
        f.write("| kernel | launches | total us | avg us | share |\n|---|---|---|---|---|\n")
        for k, (n, us) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| `{k}` | {n} | {us:.1f} | {us / n:.2f} | {us / total:.3f} |\n")
    print(open(dst).read())


def full(src, dst):
    out = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    with open(dst, "w") as f:
        f.write(f"# ncu --set full summary ({src})\n\n")
        for r in rows[2:]:
            f.write(f"## {short(r[hdr.index('Kernel Name')])}  (id {r[0]})\n\n| metric | value | unit |\n|---|---|---|\n")
            for m in FULL_METRICS:
                if m in hdr:
                    i = hdr.index(m)
                    f.write(f"| {m} | {r[i]} | {units[i]} |\n")
            f.write("\n")
    print(open(dst).read())


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 0)
    else:
        full(sys.argv[2], sys.argv[3])
