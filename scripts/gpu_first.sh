#!/bin/bash
# First GPU pass: parity tests, bench, ncu launch list, one full capture of the top kernel.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"
tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_bench.log 2>&1; echo "ncu_list_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_kernel -s 1 -c 2 -o gpurun_out/prof_match -f \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_match.log 2>&1; echo "ncu_full_rc=$?"
ls -la gpurun_out
