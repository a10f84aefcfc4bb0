cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -k back_to_back > gpurun_out/pytest_b2b.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_b2b.log
