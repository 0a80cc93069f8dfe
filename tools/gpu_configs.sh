#!/bin/bash
# Bench line per BASELINE config (full size) + a time-limited solve's KKT.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
: > gpurun_out/configs.log
for cfg in 1 3 5 4; do
  echo "== config $cfg" >> gpurun_out/configs.log
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --time-to-tol 0 --skip-cpu-baseline \
    > gpurun_out/bench_cfg$cfg.json 2> gpurun_out/bench_cfg$cfg.err
  echo "exit $?" >> gpurun_out/configs.log
  tail -2 gpurun_out/bench_cfg$cfg.err >> gpurun_out/configs.log
  python -c "import json; l=json.loads(open('gpurun_out/bench_cfg$cfg.json').readline()); print(round(l['value']), 'it/s', round(1000*l['roofline']['kernel_ms_per_trial'],2), 'us/trial', round(l['roofline']['frac'],3), l['e2e']['value'], l['config']['nnz'])" >> gpurun_out/configs.log 2>&1
done
