cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/sizes_db.log
for sh in 0 1 2; do echo "shape $sh" >> gpurun_out/sizes_db.log; GPM_DB_SHAPE=$sh timeout 600 python tools/time_d1_sizes.py 2>&1 | grep '"path": 3' >> gpurun_out/sizes_db.log; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -x -k "reduce_then_scan or large_n_sampled" > gpurun_out/pytest_big.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_big.log
