#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
export FOLP_NO_GRAPH=1
timeout 300 python tools/profile_loop.py --warmup 3 --periods 2 > gpurun_out/profile_loop.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:k_ndg_bisect' --launch-skip 2 -c 1 \
  -o gpurun_out/bisect_full -f python tools/profile_loop.py --warmup 3 --periods 2 > gpurun_out/ncu_bisect.log 2>&1
