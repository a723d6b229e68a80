#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"; tail -5 gpurun_out/bench.err
python scripts/show_bench.py gpurun_out/bench.json 2>/dev/null | head -34
DG_FORCE_SHARDED=1 timeout 900 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-profile --scale 20 --batch 200000 > gpurun_out/bench_sharded1.json 2> gpurun_out/bench_sharded1.err; echo "sharded_bench_rc=$?"; tail -5 gpurun_out/bench_sharded1.err; cut -c1-400 gpurun_out/bench_sharded1.json
