for c in 2 3 5; do FOLP_ENGINE_LIB=$PWD/variants/libfolp_bt.so FOLP_TIMING=1 timeout 300 python tools/profile_loop.py --config $c --warmup 3 --periods 10 > gpurun_out/bt${c}b.txt 2>&1; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
