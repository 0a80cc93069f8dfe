#!/bin/bash
# Warm launch list of 2 evaluation periods for config $1 (default 3).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
CFG=${1:-3}
export FOLP_NO_GRAPH=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/launches_cfg$CFG.csv python tools/profile_loop.py --config $CFG --warmup 3 --periods 2 > gpurun_out/ncu_launch_cfg$CFG.log 2>&1
