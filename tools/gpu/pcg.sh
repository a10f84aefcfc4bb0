cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/prof_pcg.py > gpurun_out/pcg.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv \
  --log-file gpurun_out/pcg_launches.csv python tools/prof_pcg.py > gpurun_out/pcg_ncu.log 2>&1
