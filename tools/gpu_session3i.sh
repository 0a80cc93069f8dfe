#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
bash tools/gpu_launches.sh
python tools/ncu_summary.py gpurun_out/launches.csv 40 > gpurun_out/launches_summary.txt 2>&1
bash tools/gpu_profile.sh
ncu -i gpurun_out/step_full.ncu-rep --page raw --csv > gpurun_out/step_full_raw.csv 2>/dev/null
