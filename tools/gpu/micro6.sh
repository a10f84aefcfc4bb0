cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 60 ./tools/micro/floor > gpurun_out/floor.log 2>&1
