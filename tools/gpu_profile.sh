#!/bin/bash
# ncu full capture (fine PC sampling) of the two step kernels (cfg2).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
export FOLP_NO_GRAPH=1
timeout 300 python tools/profile_loop.py --warmup 2 --periods 2 > gpurun_out/profile_loop.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  --warp-sampling-interval 0 --warp-sampling-max-passes 20 \
  -k 'regex:segdot_kernel<folpgpu::Epi(Primal|Dual), \(bool\)0, \(bool\)0>' --launch-skip 40 -c 2 \
  -o gpurun_out/step_full -f python tools/profile_loop.py --warmup 2 --periods 2 > gpurun_out/ncu_full.log 2>&1
