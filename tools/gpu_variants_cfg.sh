#!/bin/bash
# variants x configs: short bench of each
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
cp paper_2106_04756_b200/lib/libfolp_b200.so /tmp/keep.so
for cfg in ${CONFIGS:-2 4}; do
for v in variants/*.so; do
  cp "$v" paper_2106_04756_b200/lib/libfolp_b200.so
  echo "== cfg$cfg $v" >> gpurun_out/variants.log
  timeout 900 python bench.py --config $cfg --steps ${STEPS:-10} --warmup 3 --time-to-tol 0 --skip-cpu-baseline 2>&1 | \
    python -c "import json,sys; l=json.loads(sys.stdin.readline()); print(round(l['value'],1), round(1000*l['roofline']['kernel_ms_per_trial'],2), round(l['roofline']['frac'],3))" >> gpurun_out/variants.log 2>&1
done
done
cp /tmp/keep.so paper_2106_04756_b200/lib/libfolp_b200.so
