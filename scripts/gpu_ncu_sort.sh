#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sort_pass" -s 4 -c 1 -o gpurun_out/prof_sort -f \
  python scripts/bench_sort.py 22 16 > gpurun_out/ncu_sort.log 2>&1; echo "ncu_rc=$?"
