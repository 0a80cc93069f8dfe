#!/bin/bash
# Launch list (per-kernel durations, cold/serialized under ncu) of 2 evaluation periods, config 2.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
export FOLP_NO_GRAPH=1
timeout 300 python tools/profile_loop.py --warmup 3 --periods 2 > gpurun_out/profile_loop.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/launches.csv python tools/profile_loop.py --warmup 3 --periods 2 > gpurun_out/ncu_launch.log 2>&1
