#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
CONFIGS="1 3 5" bash tools/gpu_round.sh
CFG=2 OUT=cfg2_full SKIP=40 COUNT=2 KREGEX="segdot_kernel<folpgpu::Epi(Primal|Dual)," bash tools/gpu_profile_kernel.sh
rm -f gpurun_out/*.ncu-rep gpurun_out/*.src.csv
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --time-to-tol 0 --skip-cpu-baseline --ordered-steps 0 > gpurun_out/ncu_bench.log 2>&1
CFG=2 bash tools/gpu_warm_traffic.sh
CFG=5 SKIP=20 bash tools/gpu_warm_traffic.sh
