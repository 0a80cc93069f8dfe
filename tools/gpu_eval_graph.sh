cd /root/repo
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_shard.py tests/test_reference_kats.py -q -x -m gpu > gpurun_out/quick_pytest.log 2>&1
: > gpurun_out/ab.log
for v in 0 1; do
  for cfg in 2 1; do
    echo "== FOLP_EVAL_GRAPH=$v cfg$cfg" >> gpurun_out/ab.log
    FOLP_EVAL_GRAPH=$v FOLP_TIMING=1 timeout 120 python tools/convergence_trace.py --config $cfg --seconds 8 --every 100000000 2>&1 | grep "timing\] total" >> gpurun_out/ab.log
    FOLP_EVAL_GRAPH=$v timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --time-to-tol 0 --skip-cpu-baseline 2>&1 | python -c "import json,sys; l=json.loads(sys.stdin.readline()); print('bench', round(l['value']), round(l['ms_per_step'],3))" >> gpurun_out/ab.log 2>&1
  done
done
