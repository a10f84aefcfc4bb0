# Round evidence (part 2): one ncu --set full capture of the headline kernel (user order),
# after the same command ran clean without ncu.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/prof_apply.py --config 2 --nu2 5 --applies 5 > gpurun_out/prof.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_d1_ov -s 2 -c 1 -f \
  -o gpurun_out/r01_d1_ov_user_nu52_full python tools/prof_apply.py --config 2 --nu2 5 --applies 5 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out > gpurun_out/ls.txt
