cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/near.log
for lb in "3,8,5" "4,8,5" "5,8,5" "6,8,5"; do GPM_NEAR_LB=$lb timeout 120 python tools/sweep_near.py 3 3 >> gpurun_out/near.log 2>&1; done
for lb in "3,8,5" "4,8,5" "5,8,5"; do GPM_NEAR_LB=$lb timeout 120 python tools/sweep_near.py 5 3 1 >> gpurun_out/near.log 2>&1; done
for lb in "4,7,5" "4,8,5" "4,9,5" "4,8,4" "4,8,6" "4,7,4" "4,9,6"; do GPM_NEAR_LB=$lb timeout 200 python tools/sweep_near.py 4 5 >> gpurun_out/near.log 2>&1; done
