cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 ./tools/micro/tma_gather > gpurun_out/tma_gather.log 2>&1
timeout 300 python tools/phase_d1.py > gpurun_out/phase_d1.log 2>&1
