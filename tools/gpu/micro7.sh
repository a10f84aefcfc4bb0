cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 60 ./tools/micro/tma_gather > gpurun_out/tma_gather.log 2>&1
