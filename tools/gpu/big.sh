cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -x -k "reduce_then_scan or large_n_sampled" > gpurun_out/pytest_big.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_big.log
timeout 900 python tools/time_d1_sizes.py > gpurun_out/sizes.log 2>&1
