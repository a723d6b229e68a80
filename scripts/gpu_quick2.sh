#!/bin/bash
# quick iteration: selected parity tests + short bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"; tail -5 gpurun_out/bench.err
python scripts/show_bench.py gpurun_out/bench.json 2>/dev/null | head -40
