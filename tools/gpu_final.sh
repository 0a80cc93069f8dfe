#!/bin/bash
# Round-end measurement pass: GPU tests, bench lines of every config, the
# reference arm, step-kernel ncu captures (configs 5, 3, 2), the bench
# command's launch list (FOLP_NO_GRAPH=1 so that ncu lists the chunk
# graph's kernels), smoke, and solves to 1e-8 with the host recheck.
#   SKIP_LONG=1 leaves out config 4's bench and solve (~25 GPU-minutes).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
if [ -n "$SKIP_LONG" ]; then CONFIGS="1 3 5" bash tools/gpu_round.sh; else CONFIGS="1 3 5 4" bash tools/gpu_round.sh; fi
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
CFG=5 OUT=cfg5_full SKIP=20 COUNT=2 KREGEX="(pair_kernel<folpgpu::EpiPrimal>|segdot_kernel<folpgpu::EpiDual,)" bash tools/gpu_profile_kernel.sh
CFG=3 OUT=cfg3_full SKIP=20 COUNT=2 KREGEX="segdot_kernel<folpgpu::Epi(Primal|Dual)," bash tools/gpu_profile_kernel.sh
CFG=2 OUT=cfg2_full SKIP=40 COUNT=2 KREGEX="segdot_kernel<folpgpu::Epi(Primal|Dual)," bash tools/gpu_profile_kernel.sh
rm -f gpurun_out/*.ncu-rep gpurun_out/*.src.csv
FOLP_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --time-to-tol 0 --skip-cpu-baseline --ordered-steps 0 > gpurun_out/ncu_bench.log 2>&1
timeout 900 python tools/kkt_recheck.py --configs 1,3,5 --seconds 60,300,300 > gpurun_out/kkt_recheck.jsonl 2> gpurun_out/kkt_recheck.err
[ -n "$SKIP_LONG" ] || timeout 1500 python tools/convergence_campaign.py --configs 4 --seconds 1300 > gpurun_out/convergence_cfg4.jsonl 2> gpurun_out/convergence_cfg4.err
