#!/bin/bash
# compute-sanitizer over the round-2 kernels (fused delete, bulk-init copy, submitted ops, sharded round protocol) + soaks
mkdir -p gpurun_out
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q \
  -k "not config3 and not config1 and not rmat and not sharded and not dropin and not headline" > gpurun_out/memcheck.log 2>&1; echo "memcheck_rc=$?"; tail -4 gpurun_out/memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q \
  -k "bulk_init_fresh_pool_kernel or submitted_failure or csr_native_block_path_hubs or known_answers" > gpurun_out/racecheck.log 2>&1; echo "racecheck_rc=$?"; tail -4 gpurun_out/racecheck.log
timeout 1500 python scripts/stress_parity.py --seeds ${SEEDS:-6000} --first 3000000 > gpurun_out/stress.log 2>&1; echo "stress_rc=$?"; tail -2 gpurun_out/stress.log
timeout 1200 python scripts/stress_parity.py --hubs --seeds ${HSEEDS:-400} --first 40000 > gpurun_out/stress_hubs.log 2>&1; echo "stress_hubs_rc=$?"; tail -2 gpurun_out/stress_hubs.log
