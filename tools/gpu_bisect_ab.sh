for v in 0 4096; do
  echo "== FOLP_BISECT_SMALL=$v"
  FOLP_BISECT_SMALL=$v FOLP_TIMING=1 timeout 300 python tools/profile_loop.py --config 2 --warmup 3 --periods 10 2>&1 | grep -i "gap\|periods"
  FOLP_NO_GRAPH=1 FOLP_BISECT_SMALL=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:k_ndg_bisect --csv --log-file gpurun_out/bis_$v.csv python tools/profile_loop.py --config 2 --warmup 3 --periods 3 > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/bis_$v.csv 3
done
