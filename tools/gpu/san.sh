cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_cases.py > gpurun_out/san_memcheck.log 2>&1; echo "exit $?" >> gpurun_out/san_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_cases.py > gpurun_out/san_racecheck.log 2>&1; echo "exit $?" >> gpurun_out/san_racecheck.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_cases.py > gpurun_out/san_synccheck.log 2>&1; echo "exit $?" >> gpurun_out/san_synccheck.log
