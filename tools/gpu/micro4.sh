cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 ./tools/micro/lat > gpurun_out/lat.log 2>&1
