#!/bin/bash
# Ordered (bit-exact) reduction mode throughput probe: config 2 / 5 / 3 bench lines.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
for cfg in 2 5 3; do
  FOLP_REDUCTION=ordered timeout 600 python bench.py --config $cfg --steps 3 --warmup 1 --time-to-tol 0 --skip-cpu-baseline > gpurun_out/ord_cfg$cfg.json 2> gpurun_out/ord_cfg$cfg.err
done
tail -c 1500 gpurun_out/ord_cfg*.json
