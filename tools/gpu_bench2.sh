#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "exit $?" >> gpurun_out/bench_default.log
timeout 600 python bench.py --parallelism shards --steps 10 --warmup 3 --time-to-tol 0 --skip-cpu-baseline > gpurun_out/bench_shard1.log 2>&1; echo "exit $?" >> gpurun_out/bench_shard1.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "exit $?" >> gpurun_out/bench_ref.log
