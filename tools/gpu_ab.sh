#!/bin/bash
# A/B of engine settings via environment variables: $@ = "NAME=VALUE ..." sets
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
: > gpurun_out/ab.log
for setting in "$@"; do
  echo "== $setting" >> gpurun_out/ab.log
  env $setting timeout 300 python bench.py --steps 20 --warmup 5 --time-to-tol 0 --skip-cpu-baseline 2>&1 | \
    python -c "import json,sys; l=json.loads(sys.stdin.readline()); print(round(l['value']), round(1000*l['roofline']['kernel_ms_per_trial'],2), round(l['roofline']['frac'],3))" >> gpurun_out/ab.log 2>&1
done
