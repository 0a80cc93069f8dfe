#!/bin/bash
# Steady-state (warm L2) DRAM traffic of the step kernels: ncu WITHOUT cache
# flushes between replays (--cache-control none), a few metrics only, so a
# launch sees the L2 its own previous pass left (config ${CFG:-2}).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
export FOLP_NO_GRAPH=1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
  --clock-control none --cache-control none --kernel-name-base demangled \
  -k "regex:(pair_kernel|segdot_kernel)<folpgpu::Epi(Primal|Dual)[,>]" --launch-skip ${SKIP:-40} -c ${COUNT:-6} --csv \
  --log-file gpurun_out/warm_traffic_cfg${CFG:-2}.csv python tools/profile_loop.py --config ${CFG:-2} --warmup 2 --periods 1 \
  > gpurun_out/warm_traffic_cfg${CFG:-2}.log 2>&1
