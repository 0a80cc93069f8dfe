cd /root/repo
: > gpurun_out/ab.log
for w in 2097152 4194304 8388608; do
  echo "== window $w" >> gpurun_out/ab.log
  FOLP_GATHER_WINDOW=$w timeout 900 python bench.py --config 4 --steps 6 --warmup 2 --time-to-tol 0 --skip-cpu-baseline 2>&1 | \
    python -c "import json,sys; l=json.loads(sys.stdin.readline()); print(round(l['value'],1), round(1000*l['roofline']['kernel_ms_per_trial'],2), round(l['roofline']['frac'],3), round(l['e2e']['value'],1))" >> gpurun_out/ab.log 2>&1
done
