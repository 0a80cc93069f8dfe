#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out; rm -f gpurun_out/hot_ab3.txt
nproc > gpurun_out/nproc.txt
for v in 1 0 1 0; do
  FOLP_HOT_COLUMNS=$v FOLP_TIMING=1 timeout 300 python bench.py --steps 20 --warmup 3 --time-to-tol 0 --skip-cpu-baseline > gpurun_out/hot_bench_$v.json 2> gpurun_out/hot_bench_$v.err
  python -c "import json; d=json.load(open('gpurun_out/hot_bench_$v.json')); print('hot=$v value', round(d['value']), 'trial_us', round(d['roofline']['kernel_ms_per_trial']*1e3,2), 'e2e', round(d['e2e']['value']), d['e2e']['seconds'])" >> gpurun_out/hot_ab3.txt
  grep -h "setup stages" gpurun_out/hot_bench_$v.err | tail -1 >> gpurun_out/hot_ab3.txt
done
