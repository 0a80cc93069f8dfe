#!/bin/bash
# A switch that must not change a bit: tools/solve_hash.py lines per setting
# ("NAME=V" arguments; plus one with no override), then the bench A/B.
#   bash tools/gpu_ab_bits.sh FOLP_DEFER_A=0
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
: > gpurun_out/ab_bits.txt
for setting in base "$@"; do
  envs=()
  [ "$setting" != base ] && IFS=, read -ra envs <<< "$setting"
  for c in "2 1.0" "3 0.2" "5 0.2" "1 1.0"; do set -- $c
    env "${envs[@]}" timeout 300 python tools/solve_hash.py --config $1 --scale $2 2>&1 | tail -1 | sed "s/^/$setting: /" >> gpurun_out/ab_bits.txt
  done
done
cat gpurun_out/ab_bits.txt
