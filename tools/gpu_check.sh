#!/bin/bash
# GPU check: tests, timing breakdown of a few solves, short bench.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/box.txt 2>&1
timeout 300 python tools/diag_restarts.py > gpurun_out/diag.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for cfg in 1 2; do
  FOLP_TIMING=1 timeout 300 python tools/convergence_trace.py --config $cfg --seconds 20 --every 1000000 \
    > gpurun_out/timing_cfg$cfg.log 2>&1
done
timeout 600 python bench.py --steps 20 --warmup 5 --time-to-tol 0 > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
