#!/bin/bash
# Microbench ceilings + ncu full capture of the two step kernels (cfg2).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
: timeout 300 ./tools/microbench/spmv_ceiling 2 > gpurun_out/ceiling.log 2>&1
export FOLP_NO_GRAPH=1
timeout 300 python tools/profile_loop.py --warmup 2 --periods 2 > gpurun_out/profile_loop.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:segpipe_kernel<folpgpu::Epi(Primal|Dual)>' --launch-skip 40 -c 4 \
  -o gpurun_out/step_full -f python tools/profile_loop.py --warmup 2 --periods 2 > gpurun_out/ncu_full.log 2>&1
: timeout 300 python tools/diag_restarts.py > gpurun_out/diag.log 2>&1
