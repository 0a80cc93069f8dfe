#!/bin/bash
# A/B of two engine builds (FOLP_ENGINE_LIB): the in-tree library vs
# ab/libfolp_b200_prev.so, per config: bench value + duality-gap pass counts.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
: > gpurun_out/ab_lib.log
for cfg in ${CONFIGS:-2 5}; do
  for lib in paper_2106_04756_b200/lib/libfolp_b200.so ab/libfolp_b200_prev.so; do
    for rep in 1 2; do
      echo "== cfg$cfg $lib rep$rep" >> gpurun_out/ab_lib.log
      FOLP_ENGINE_LIB=$PWD/$lib FOLP_TIMING=1 timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 \
        --time-to-tol 0 --skip-cpu-baseline 2> gpurun_out/ab_err.log | \
        python -c "import json,sys; l=json.loads(sys.stdin.readline()); print(round(l['value']), l['ms_per_step'])" >> gpurun_out/ab_lib.log 2>&1
      grep "duality gaps" gpurun_out/ab_err.log | tail -2 >> gpurun_out/ab_lib.log
    done
  done
done
