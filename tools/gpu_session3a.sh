cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/box.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
CONFIGS="2 3 5" bash tools/gpu_ab.sh FOLP_DYN_FRAC=0 FOLP_DYN_FRAC=0.1 FOLP_DYN_FRAC=0.35 > gpurun_out/ab_dyn.txt 2>&1
