#!/bin/bash
# Round 2 first pass: parity tests, two soaks, bench.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python scripts/stress_parity.py --seeds ${SEEDS:-400} > gpurun_out/stress.log 2>&1; echo "stress_rc=$?"; tail -3 gpurun_out/stress.log
timeout 900 python scripts/stress_parity.py --hubs --seeds ${HSEEDS:-60} > gpurun_out/stress_hubs.log 2>&1; echo "stress_hubs_rc=$?"; tail -3 gpurun_out/stress_hubs.log
timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"
tail -5 gpurun_out/bench.err
python scripts/show_bench.py gpurun_out/bench.json
