#!/bin/bash
# Warm launch lists (ncu gpu__time_duration, --cache-control none) of one
# evaluation period of config ${CFG:-2}, one per "NAME=V" argument.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
export FOLP_NO_GRAPH=1
for setting in "$@"; do
  tag=$(echo "$setting" | tr ',=' '__')
  env $setting timeout 300 python tools/profile_loop.py --config ${CFG:-2} --warmup 3 --periods 1 > gpurun_out/pl_$tag.log 2>&1 || continue
  env $setting timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/launches_$tag.csv python tools/profile_loop.py --config ${CFG:-2} --warmup 3 --periods 1 > gpurun_out/ncu_$tag.log 2>&1
  python tools/ncu_summary.py gpurun_out/launches_$tag.csv 12 > gpurun_out/launches_$tag.txt 2>&1
  echo "== $setting"; cat gpurun_out/launches_$tag.txt
done
