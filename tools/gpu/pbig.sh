cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/prof_big.py > gpurun_out/pbig.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
  --log-file gpurun_out/pbig_launches.csv python tools/prof_big.py > gpurun_out/pbig_ncu.log 2>&1
