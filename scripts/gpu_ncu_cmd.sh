#!/bin/bash
# usage: KREGEX=<regex> SKIP=<n> COUNT=<n> NAME=<out> CMD="python ..." bash scripts/gpu_ncu_cmd.sh
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s ${SKIP:-2} -c ${COUNT:-1} -o gpurun_out/${NAME:-prof} -f \
  ${CMD} > gpurun_out/ncu_${NAME:-prof}.log 2>&1; echo "ncu_full_rc=$?"
tail -1 gpurun_out/ncu_${NAME:-prof}.log | cut -c1-200
