#!/bin/bash
# e2e breakdown after the threaded histogram (config 2, 800 iterations, FOLP_TIMING).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
FOLP_TIMING=1 timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e_breakdown.txt 2>&1
for i in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 3 --time-to-tol 0 --skip-cpu-baseline > gpurun_out/e2e_bench_$i.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2e_bench_$i.json')); print('value', round(d['value']), 'e2e', round(d['e2e']['value']), d['e2e']['seconds'])" >> gpurun_out/e2e_breakdown.txt
done
