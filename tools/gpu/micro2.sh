cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 ./tools/micro/tma_gather > gpurun_out/tma_gather.log 2>&1
timeout 120 ./tools/micro/icache > gpurun_out/icache.log 2>&1
