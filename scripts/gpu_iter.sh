#!/bin/bash
# Iteration pass: parity tests, bench (no cpu baseline), optional extras via env.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_rc=$?"
tail -15 gpurun_out/pytest_gpu.log
if [ "${SANITIZE:-0}" = "1" ]; then
  timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "known_answers_vs_oracle" > gpurun_out/memcheck.log 2>&1; echo "memcheck_rc=$?"
  tail -5 gpurun_out/memcheck.log
fi
timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"
tail -5 gpurun_out/bench.err
python scripts/show_bench.py gpurun_out/bench.json
