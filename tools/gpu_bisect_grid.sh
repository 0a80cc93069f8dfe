#!/bin/bash
# Duality-gap bisection: pass statistics and per-launch time per cooperative grid size.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
for g in ${GRIDS:-296 148 74}; do
  echo "== FOLP_BISECT_GRID=$g"
  FOLP_BISECT_GRID=$g FOLP_TIMING=1 timeout 300 python tools/profile_loop.py --config ${CFG:-2} --warmup 3 --periods 10 2>&1 | grep -i "gap\|periods"
  FOLP_NO_GRAPH=1 FOLP_BISECT_GRID=$g timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ndg_bisect --csv --log-file gpurun_out/bisg_$g.csv python tools/profile_loop.py --config ${CFG:-2} --warmup 3 --periods 3 > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/bisg_$g.csv 3
done
