cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/sweep_d1.py 4 > gpurun_out/sweep.log 2>&1
timeout 600 python tools/prof_apply.py --config 2 --nu2 5 --applies 3 --rank --nrhs 16 > gpurun_out/prof16.log 2>&1
timeout 900 python bench.py --no-cpu --steps 500 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
