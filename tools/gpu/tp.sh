cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/time_predict.py > gpurun_out/tp.log 2>&1
