#!/bin/bash
# After an engine change: GPU tests, short benches of configs 2/5/3, the
# config-2 launch list (ncu, after the same program ran clean without it).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
for cfg in ${CONFIGS:-2 5 3}; do
  timeout 600 python bench.py --config $cfg --steps 20 --warmup 3 --time-to-tol 0 --skip-cpu-baseline \
    > gpurun_out/verify_cfg$cfg.json 2> gpurun_out/verify_cfg$cfg.err
done
bash tools/gpu_launches.sh
