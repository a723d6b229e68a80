#!/bin/bash
# Quick iteration: selected GPU tests (K=pytest -k expr) then a short bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${K:+-k "$K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_rc=$?"
tail -${TAIL:-15} gpurun_out/pytest_gpu.log
if [ "${BENCH:-1}" = "1" ]; then
timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"
tail -5 gpurun_out/bench.err
python scripts/show_bench.py gpurun_out/bench.json
fi
