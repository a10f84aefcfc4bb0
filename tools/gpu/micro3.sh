cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 ./tools/micro/icache > gpurun_out/icache.log 2>&1
