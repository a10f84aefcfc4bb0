# Round evidence: GPU tests, smoke, bench line, ncu launch list of the bench command, one
# ncu --set full capture of the headline kernel (each ncu pass after its command ran clean).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-extras --no-cpu > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_bench_small.csv python bench.py --steps 20 --warmup 3 --no-extras --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/prof_apply.py --config 2 --nu2 5 --applies 5 > gpurun_out/prof.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_d1_ov -s 2 -c 1 -f \
  -o gpurun_out/r01_d1_ov_user_nu52_full python tools/prof_apply.py --config 2 --nu2 5 --applies 5 > gpurun_out/ncu_full.log 2>&1
