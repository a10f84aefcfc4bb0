#!/bin/bash
# One driver for every gpurun evidence pass (run from the repo root on the GPU box):
#   gpurun --timeout T -- 'bash tools/gpu/run.sh <task> [args]; bash tools/gpu/run.sh <task2> ...'
# tasks (outputs under gpurun_out/, one log per task):
#   tests [pytest args]   pytest -m gpu (default -x -q)
#   smoke                 __graft_entry__.smoke()
#   bench [bench args]    bench.py (clocks are sampled inside bench.py)
#   launches [args]       plain bench run, then the ncu launch list of the same command
#   full <regex> [args]   plain bench run, then one ncu --set full capture of kernels matching <regex>
#   sanitize <tool>       compute-sanitizer --tool <tool> over tools/sanitize_cases.py
#   py <script> [args]    any python script (timing tools under tools/)
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
task=${1:-tests}
shift || true
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv \
  > "gpurun_out/smi_$task.txt" 2>&1
case "$task" in
  tests)
    timeout 2400 python -m pytest tests -m gpu ${@:--x -q} > gpurun_out/pytest_gpu.log 2>&1
    echo "pytest exit $?" >> gpurun_out/pytest_gpu.log ;;
  smoke)
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
    echo "smoke exit $?" >> gpurun_out/smoke.log ;;
  bench)
    timeout 900 python bench.py "$@" > gpurun_out/bench.log 2>&1
    echo "bench exit $?" >> gpurun_out/bench.log ;;
  launches)
    timeout 900 python bench.py "$@" > gpurun_out/launches_plain.log 2>&1 &&
    timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py "$@" \
      > gpurun_out/launches_ncu.log 2>&1
    echo "launches exit $?" >> gpurun_out/launches_ncu.log ;;
  full)
    rx=$1
    shift
    timeout 900 python bench.py "$@" > gpurun_out/full_plain.log 2>&1 &&
    timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$rx" -s 3 -c 1 \
      -o gpurun_out/full python bench.py "$@" > gpurun_out/full_ncu.log 2>&1
    echo "full exit $?" >> gpurun_out/full_ncu.log ;;
  sanitize)
    tool=$1
    timeout 1500 compute-sanitizer --tool "$tool" --print-limit 20 python tools/sanitize_cases.py \
      > "gpurun_out/san_$tool.log" 2>&1
    echo "exit $?" >> "gpurun_out/san_$tool.log" ;;
  py)
    s=$1
    shift
    b=$(basename "$s" .py)
    timeout 1500 python "$s" "$@" > "gpurun_out/py_$b.log" 2>&1
    echo "exit $?" >> "gpurun_out/py_$b.log" ;;
  *) echo "unknown task $task" >&2; exit 2 ;;
esac
