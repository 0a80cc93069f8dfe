#!/bin/bash
# Session 3: gap setup from the convergence_info K'y (A/B against FOLP_NDG_RAW=1), GPU tests.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
for c in 2 3 5; do
  for v in new old; do
    if [ $v = old ]; then export FOLP_NDG_RAW=1; else unset FOLP_NDG_RAW; fi
    echo "cfg$c $v: $(FOLP_TIMING=1 timeout 300 python tools/profile_loop.py --config $c --warmup 3 --periods 10 2>&1 | grep -E 'periods:|duality gaps')"
  done
done > gpurun_out/ndgraw_ab.txt 2>&1
unset FOLP_NDG_RAW
CONFIGS="2" bash tools/gpu_ab.sh FOLP_NDG_RAW=1 >> gpurun_out/ndgraw_ab.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
