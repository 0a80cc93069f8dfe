#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 1200 ./tools/microbench/spmv_ceiling 4 1.0 > gpurun_out/ceiling4.log 2>&1
