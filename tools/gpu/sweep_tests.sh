cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/sweep_d1.py 2 4 > gpurun_out/sweep.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
