#!/bin/bash
# usage: KREGEX=<regex> SKIP=<n> COUNT=<n> NAME=<out> bash scripts/gpu_ncu_full.sh
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s ${SKIP:-2} -c ${COUNT:-2} -o gpurun_out/${NAME:-prof} -f \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_${NAME:-prof}.log 2>&1; echo "ncu_full_rc=$?"
tail -1 gpurun_out/ncu_${NAME:-prof}.log | cut -c1-200
