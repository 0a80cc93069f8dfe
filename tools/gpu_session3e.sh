#!/bin/bash
# Session 3: column renumbering (sort-free, threaded) -- GPU tests, bench A/B with e2e.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
for v in 1 0 1 0; do
  FOLP_HOT_COLUMNS=$v FOLP_TIMING=1 timeout 300 python bench.py --steps 20 --warmup 3 --time-to-tol 0 --skip-cpu-baseline > gpurun_out/hot_bench_$v.json 2> gpurun_out/hot_bench_$v.err
  python -c "import json; d=json.load(open('gpurun_out/hot_bench_$v.json')); print('hot=$v value', round(d['value']), 'trial_us', round(d['roofline']['kernel_ms_per_trial']*1e3,2), 'e2e', round(d['e2e']['value']), d['e2e']['seconds'])" >> gpurun_out/hot_ab2.txt
  grep -h "setup stages" gpurun_out/hot_bench_$v.err | tail -1 >> gpurun_out/hot_ab2.txt
done
