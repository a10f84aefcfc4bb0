cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/sweep_d1.py 4 > gpurun_out/sweep.log 2>&1
GPM_D1_SHAPE=4 timeout 300 python tools/phase_d1.py > gpurun_out/phase4.log 2>&1
GPM_D1_SHAPE=7 timeout 300 python tools/phase_d1.py > gpurun_out/phase7.log 2>&1
