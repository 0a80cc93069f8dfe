#!/bin/bash
# Round-end style check: GPU tests, default bench, reference arm, other configs.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/box.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "exit $?" >> gpurun_out/bench_default.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for cfg in ${CONFIGS:-1 3 5 4}; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --time-to-tol 0 --skip-cpu-baseline > gpurun_out/bench_cfg$cfg.json 2> gpurun_out/bench_cfg$cfg.err
done
