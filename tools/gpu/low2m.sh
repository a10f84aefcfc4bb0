cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/engine_ab.py > gpurun_out/engine_ab.log 2>&1
GPM_LOW2_PERCOL=1 timeout 300 python tools/engine_ab.py 0,1 > gpurun_out/engine_ab_percol.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
