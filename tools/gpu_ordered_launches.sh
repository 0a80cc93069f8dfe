#!/bin/bash
# Launch list of ordered (bit-exact) mode, config 2: 1 warm-up + 1 evaluation period.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
export FOLP_REDUCTION=ordered FOLP_NO_GRAPH=1
timeout 300 python tools/profile_loop.py --warmup 1 --periods 1 > gpurun_out/ol_profile_loop.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/ol_launches.csv python tools/profile_loop.py --warmup 1 --periods 1 > gpurun_out/ol_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/ol_launches.csv 25
