#!/bin/bash
# Session 3: column renumbering -- GPU tests, bench A/B (FOLP_HOT_COLUMNS=0 vs default) on configs 2 3 5.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
CONFIGS="2" bash tools/gpu_ab.sh FOLP_HOT_COLUMNS=0 > gpurun_out/hot_ab.txt 2>&1
for v in 1 0; do
  FOLP_HOT_COLUMNS=$v FOLP_TIMING=1 timeout 300 python bench.py --steps 5 --warmup 3 --time-to-tol 0 --skip-cpu-baseline > gpurun_out/hot_bench_$v.json 2> gpurun_out/hot_bench_$v.err
done
