#!/bin/bash
# Exact-fold session 2: fold tests + ordered launch list (config 2).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_exact_fold.py -x -q -s > gpurun_out/e2_fold.log 2>&1; echo "exit $?" >> gpurun_out/e2_fold.log
tail -5 gpurun_out/e2_fold.log
export FOLP_REDUCTION=ordered FOLP_NO_GRAPH=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_exact_fold|segdot_kernel<Epi(Primal|Dual)," \
  --log-file gpurun_out/e2_launches.csv python tools/profile_loop.py --warmup 0 --periods 1 > gpurun_out/e2_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/e2_launches.csv 10
