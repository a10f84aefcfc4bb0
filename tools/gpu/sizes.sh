cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/time_d1_sizes.py > gpurun_out/sizes.log 2>&1
