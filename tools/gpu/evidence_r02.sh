#!/bin/bash
# Round-2 evidence passes (run from the repo root on the GPU box; outputs under gpurun_out/,
# text only: the .ncu-rep files are summarised there and removed -- gpurun returns <= 64 MiB):
#   bash tools/gpu/evidence_r02.sh fp64       FP64 instruction counts + DRAM bytes per apply, configs 3-5
#   bash tools/gpu/evidence_r02.sh full       ncu --set full of the d >= 2 kernels (details + per-line stalls)
#   bash tools/gpu/evidence_r02.sh launches   ncu launch list of the bench command
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
case "${1:-fp64}" in
  fp64)
    M=sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
    for spec in "3 3 0 1" "4 5 0 1" "5 3 1 1" "5 3 1 4"; do
      set -- $spec
      python tools/prof_apply.py --config $1 --nu2 $2 --form $3 --nrhs $4 --applies 2 > /dev/null 2>&1 || echo "plain run failed $spec"
      ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r02_fp64_config$1_rhs$4.csv \
        python tools/prof_apply.py --config $1 --nu2 $2 --form $3 --nrhs $4 --applies 2 > gpurun_out/fp64_$1_$4.log 2>&1
    done ;;
  full)
    python tools/prof_apply.py --config 4 --nu2 5 --applies 3 > /dev/null 2>&1
    ncu --set full --clock-control none --import-source on -k 'regex:k_mid3|k_low3|k_cp<' -s 4 -c 4 -o gpurun_out/d3 \
      python tools/prof_apply.py --config 4 --nu2 5 --applies 3 > gpurun_out/full_d3.log 2>&1
    ncu -i gpurun_out/d3.ncu-rep --page details > gpurun_out/r02_d3_config4_details.txt 2>&1
    python tools/ncu_lines.py gpurun_out/d3.ncu-rep 200 > gpurun_out/r02_d3_config4_lines.txt 2>&1
    rm -f gpurun_out/d3.ncu-rep
    python tools/prof_apply.py --config 3 --nu2 3 --applies 3 > /dev/null 2>&1
    ncu --set full --clock-control none --import-source on -k 'regex:k_low2|k_cp<' -s 3 -c 3 -o gpurun_out/d2 \
      python tools/prof_apply.py --config 3 --nu2 3 --applies 3 > gpurun_out/full_d2.log 2>&1
    ncu -i gpurun_out/d2.ncu-rep --page details > gpurun_out/r02_d2_config3_details.txt 2>&1
    rm -f gpurun_out/d2.ncu-rep ;;
  d1)
    # the headline kernel: plain run, launch list (time + DRAM bytes), one --set full capture
    B="--steps 20 --warmup 3 --no-extras --no-cpu --no-cg"
    python bench.py $B > gpurun_out/d1_plain.log 2>&1 &&
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/r02_launches_bench_d1_final.csv python bench.py $B > gpurun_out/d1_launches.log 2>&1
    ncu --set full --clock-control none --import-source on -k regex:k_d1_lpc -s 30 -c 1 -o gpurun_out/d1full \
      python bench.py $B > gpurun_out/d1_full.log 2>&1
    ncu -i gpurun_out/d1full.ncu-rep --page details > gpurun_out/r02_d1_lpc_user_full_details_final.txt 2>&1
    python tools/ncu_lines.py gpurun_out/d1full.ncu-rep 100 > gpurun_out/r02_d1_lpc_user_lines_final.txt 2>&1
    rm -f gpurun_out/d1full.ncu-rep ;;
  launches)
    python bench.py --steps 20 --warmup 3 --no-cg --no-cpu > gpurun_out/launches_plain.log 2>&1 &&
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/launches_all.csv python bench.py --steps 20 --warmup 3 --no-cg --no-cpu > gpurun_out/launches_ncu.log 2>&1
    # keep the library's own kernels (the setup's CUB sort launches are thousands of lines)
    grep -E '^"ID"|gpm::|lpc::' gpurun_out/launches_all.csv > gpurun_out/r02_launches_bench_final.csv
    rm -f gpurun_out/launches_all.csv ;;
esac
echo done
