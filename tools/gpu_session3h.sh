#!/bin/bash
# Session 3 closing check: GPU tests, smoke, default bench + reference arm.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for cfg in 3 5; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --time-to-tol 0 --skip-cpu-baseline > gpurun_out/bench_cfg$cfg.json 2> gpurun_out/bench_cfg$cfg.err
done
