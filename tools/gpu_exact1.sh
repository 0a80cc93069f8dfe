#!/bin/bash
# Exact-fold session: fold tests, ordered-mode parity (bit-exact suite), ordered-mode config-2 bench.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_exact_fold.py -x -q -s > gpurun_out/e1_fold.log 2>&1; echo "exit $?" >> gpurun_out/e1_fold.log
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_edge_cases.py tests/test_golden.py -x -q -m gpu > gpurun_out/e1_solve.log 2>&1; echo "exit $?" >> gpurun_out/e1_solve.log
FOLP_REDUCTION=ordered timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --time-to-tol 0 --skip-cpu-baseline > gpurun_out/e1_ord_cfg2.json 2> gpurun_out/e1_ord_cfg2.err
timeout 900 python -m pytest tests/test_gpu_fullsize_parity.py -x -q -s -k "2" > gpurun_out/e1_full2.log 2>&1; echo "exit $?" >> gpurun_out/e1_full2.log
tail -5 gpurun_out/e1_fold.log gpurun_out/e1_solve.log gpurun_out/e1_full2.log; tail -c 1200 gpurun_out/e1_ord_cfg2.json
