cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_robust.py -q > gpurun_out/pytest_robust.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_robust.log
