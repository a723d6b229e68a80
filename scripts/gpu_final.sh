#!/bin/bash
# Final artefacts of the round: parity tests, bench (cpu baseline + parity block), reference arm, C3, C1, C5, sort, ncu launch list, ncu full.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"; tail -3 gpurun_out/bench.err
python scripts/show_bench.py gpurun_out/bench.json | head -40
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref_rc=$?"; cut -c1-300 gpurun_out/bench_ref.json
timeout 900 python bench.py --scale 24 --batch 10000000 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3_rc=$?"; tail -3 gpurun_out/bench_c3.err
python scripts/show_bench.py gpurun_out/bench_c3.json | head -34
timeout 900 python bench.py --scale 24 --batch 10000000 --steps 5 --warmup 3 --no-cpu-baseline --pool-initial-fraction 0.4 > gpurun_out/bench_c3_grow.json 2> gpurun_out/bench_c3_grow.err; echo "c3grow_rc=$?"
timeout 900 python bench.py --block-size 0 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_b0.json 2> gpurun_out/bench_b0.err; echo "b0_rc=$?"
python scripts/show_bench.py gpurun_out/bench_b0.json | head -9
timeout 600 python scripts/bench_c1.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo "c1_rc=$?"; cut -c1-400 gpurun_out/bench_c1.json
timeout 900 python scripts/bench_mixed.py > gpurun_out/mixed_c5.json 2> gpurun_out/mixed_c5.err; echo "c5_rc=$?"; cut -c1-400 gpurun_out/mixed_c5.json
timeout 600 python scripts/bench_sort.py 22 16 > gpurun_out/sort.log 2>&1; echo "sort_rc=$?"; tail -5 gpurun_out/sort.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_bench.log 2>&1; echo "ncu_list_rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"fused_delete|group_count|append_entries|alloc_kernel|group_scatter|op_arm|match_long" -s 14 -c 12 -o gpurun_out/prof_step -f \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_step.log 2>&1; echo "ncu_full_rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"csr_bulk|csr_plan" -c 2 -o gpurun_out/prof_bulk -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/ncu_bulk.log 2>&1; echo "ncu_bulk_rc=$?"
