#!/bin/bash
# variants: timing split of a 10 s cfg2 solve + short bench each
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
cp paper_2106_04756_b200/lib/libfolp_b200.so /tmp/keep.so
for v in variants/*.so; do
  cp "$v" paper_2106_04756_b200/lib/libfolp_b200.so
  echo "== $v" >> gpurun_out/variants.log
  FOLP_TIMING=1 timeout 300 python tools/convergence_trace.py --config 2 --seconds 10 --every 100000000 2>&1 | grep -v "^it " >> gpurun_out/variants.log
  timeout 300 python bench.py --steps 20 --warmup 5 --time-to-tol 0 --skip-cpu-baseline 2>&1 | \
    python -c "import json,sys; l=json.loads(sys.stdin.readline()); print('bench', round(l['value']), round(1000*l['roofline']['kernel_ms_per_trial'],2))" >> gpurun_out/variants.log 2>&1
done
cp /tmp/keep.so paper_2106_04756_b200/lib/libfolp_b200.so
