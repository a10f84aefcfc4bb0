cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/time_d1_sizes.py > gpurun_out/sizes.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
