#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"csr_bulk|csr_plan" -c 2 -o gpurun_out/prof_bulk -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_bulk.log 2>&1; echo "ncu_rc=$?"
