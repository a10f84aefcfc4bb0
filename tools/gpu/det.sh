cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/det_check.py > gpurun_out/det.log 2>&1
