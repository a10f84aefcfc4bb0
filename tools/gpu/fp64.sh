# FP64 work per apply (d = 1, 2, 3) for the ALU roofline: thread-level DFMA / DADD / DMUL
# counts and durations per kernel from ncu (cold, serialised launches).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in "2 5 0" "3 3 0" "4 5 0" "5 3 1"; do
  set -- $c
  timeout 300 python tools/prof_apply.py --config $1 --nu2 $2 --form $3 --applies 2 > /dev/null 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/fp64_config$1.csv \
    python tools/prof_apply.py --config $1 --nu2 $2 --form $3 --applies 2 > /dev/null 2>&1
done
timeout 300 python tools/prof_apply.py --config 5 --nu2 3 --form 1 --applies 2 --rank --nrhs 4 > /dev/null 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/fp64_config5_rhs4.csv \
  python tools/prof_apply.py --config 5 --nu2 3 --form 1 --applies 2 --rank --nrhs 4 > /dev/null 2>&1
ls -la gpurun_out/fp64* > gpurun_out/fp64_ls.txt
