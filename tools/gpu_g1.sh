cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/g1_box.txt 2>&1
nproc >> gpurun_out/g1_box.txt; free -g >> gpurun_out/g1_box.txt; lscpu | head -20 >> gpurun_out/g1_box.txt
(time timeout 900 oracle/_ref/dropin/folp_acceptance) > gpurun_out/g1_accept.log 2>&1; echo "exit $?" >> gpurun_out/g1_accept.log
(time timeout 900 oracle/_ref/dropin/folp_tests) > gpurun_out/g1_units.log 2>&1; echo "exit $?" >> gpurun_out/g1_units.log
timeout 600 python bench.py > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err
tail -3 gpurun_out/g1_accept.log gpurun_out/g1_units.log; cat gpurun_out/g1_bench.json
