#!/bin/bash
# ncu --set full of kernels matching $KREGEX (demangled), config ${CFG:-2},
# with the environment given as arguments (e.g. FOLP_TWO_PHASE=1).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
export FOLP_NO_GRAPH=1
OUT=${OUT:-kernel_full}
env "$@" timeout 300 python tools/profile_loop.py --config ${CFG:-2} --warmup 2 --periods 1 > gpurun_out/$OUT.pl.log 2>&1 || exit 1
env "$@" timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:${KREGEX}" --launch-skip ${SKIP:-40} -c ${COUNT:-2} \
  -o gpurun_out/$OUT -f python tools/profile_loop.py --config ${CFG:-2} --warmup 2 --periods 1 > gpurun_out/$OUT.ncu.log 2>&1
ncu -i gpurun_out/$OUT.ncu-rep --page raw --csv > gpurun_out/$OUT.raw.csv 2>/dev/null
ncu -i gpurun_out/$OUT.ncu-rep --page source --csv --print-source sass > gpurun_out/$OUT.src.csv 2>/dev/null
ncu -i gpurun_out/$OUT.ncu-rep --page details --csv > gpurun_out/$OUT.details.csv 2>/dev/null
