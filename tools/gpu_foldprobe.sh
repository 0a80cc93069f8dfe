#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
export FOLP_FOLD_TIMES=1
timeout 300 python -m pytest tests/test_gpu_exact_fold.py -x -q -s -k speed 2>&1 | tail -5
FOLP_REDUCTION=ordered timeout 300 python -c "
from paper_2106_04756_b200 import cabi, engine, instances
lp = instances.generate(2, 1, 1.0)
eng = engine()
eng.lib.folp_gpu_set_default_reduction(1)
r = eng.solve_lp(lp, cabi.params(iteration_limit=30))
print(r.iterations)
" 2>&1 | tail -3
