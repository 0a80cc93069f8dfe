#!/bin/bash
# Exact-fold session 4: fold tests, ordered bit-exact suites, full-size parity (all configs), ordered bench.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
export FOLP_FOLD_TIMES=1
timeout 600 python -m pytest tests/test_gpu_exact_fold.py -x -q -s > gpurun_out/e4_fold.log 2>&1; echo "exit $?" >> gpurun_out/e4_fold.log
tail -4 gpurun_out/e4_fold.log
timeout 1200 python -m pytest tests/test_gpu_solve.py tests/test_gpu_edge_cases.py tests/test_golden.py tests/test_gpu_kernels.py -x -q -m gpu > gpurun_out/e4_solve.log 2>&1; echo "exit $?" >> gpurun_out/e4_solve.log
tail -4 gpurun_out/e4_solve.log
FOLP_REDUCTION=ordered timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --time-to-tol 0 --skip-cpu-baseline > gpurun_out/e4_ord_cfg2.json 2> gpurun_out/e4_ord_cfg2.err
python -c "import json; d=json.load(open('gpurun_out/e4_ord_cfg2.json')); print('ordered cfg2', d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_trial'])"
timeout 2400 python -m pytest tests/test_gpu_fullsize_parity.py -x -q -s > gpurun_out/e4_full.log 2>&1; echo "exit $?" >> gpurun_out/e4_full.log
grep -E "config|passed|failed|Error|exit" gpurun_out/e4_full.log | tail -12
