cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 60 ./tools/micro/xchg > gpurun_out/xchg.log 2>&1
