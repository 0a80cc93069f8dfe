#!/bin/bash
# Quick GPU loop: kernel tests, bench line, timing split of a cfg2 solve.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solve.py -q -x -k "not tree_mode_solve" > gpurun_out/quick_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/quick_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --time-to-tol 0 > gpurun_out/quick_bench.log 2>&1
FOLP_TIMING=1 timeout 300 python tools/convergence_trace.py --config 2 --seconds 10 --every 1000000 > gpurun_out/quick_timing.log 2>&1
