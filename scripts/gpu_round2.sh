#!/bin/bash
# Round-2 artefacts: parity tests, bench (with cpu baseline), reference arm, C3 bench, ncu launch list, ncu full of the top kernels.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"; tail -3 gpurun_out/bench.err
python scripts/show_bench.py gpurun_out/bench.json | head -30
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref_rc=$?"; cut -c1-300 gpurun_out/bench_ref.json
timeout 900 python bench.py --scale 24 --batch 10000000 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3_rc=$?"; tail -3 gpurun_out/bench_c3.err
python scripts/show_bench.py gpurun_out/bench_c3.json | head -30
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_bench.log 2>&1; echo "ncu_list_rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"fused_delete|group_count|append_entries|alloc_kernel|group_scatter" -s 12 -c 10 -o gpurun_out/prof_step -f \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_step.log 2>&1; echo "ncu_full_rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"csr_append|csr_plan" -c 2 -o gpurun_out/prof_csr -f \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_csr.log 2>&1; echo "ncu_csr_rc=$?"
