cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/sweep_sizes.py > gpurun_out/sweep_sizes.log 2>&1
