cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/micro/pcie.py > gpurun_out/pcie.log 2>&1
