#!/bin/bash
# A/B of engine switches: one bench line per "NAME=V[,NAME2=V2]" argument
# (and one with no override), for each config in $CONFIGS (default 2).
#   bash tools/gpu_ab.sh FOLP_TWO_PHASE=0 FOLP_TWO_PHASE=1
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
for cfg in ${CONFIGS:-2}; do
  for setting in base "$@"; do
    envs=()
    [ "$setting" != base ] && IFS=, read -ra envs <<< "$setting"
    tag=$(echo "$setting" | tr ',=' '__')
    env "${envs[@]}" timeout 600 python bench.py --config $cfg --steps ${STEPS:-20} --warmup 3 \
      --time-to-tol 0 --skip-cpu-baseline > gpurun_out/ab_cfg${cfg}_$tag.json 2> gpurun_out/ab_cfg${cfg}_$tag.err
    echo "cfg$cfg $setting: $(python -c "import json,sys; d=json.load(open('gpurun_out/ab_cfg${cfg}_$tag.json')); r=d['roofline']; print(round(d['value'],1), 'it/s; trial', round(r['kernel_ms_per_trial']*1000,2), 'us; frac', round(r['frac'],3))" 2>&1)"
  done
done
