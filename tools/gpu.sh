#!/bin/bash
# One entry point for GPU-box work (run from the repo root under gpurun):
#   tools/gpu.sh tests [pytest -k expr]      -m gpu suite (optionally a subset)
#   tools/gpu.sh bench TAG [bench args]      one bench line -> gpurun_out/bench_TAG.json
#   tools/gpu.sh launches TAG                ncu launch list of one timed step (tools/launch_list.sh)
#   tools/gpu.sh ncu TAG REGEX SKIP COUNT    ncu --set full of COUNT launches of kernels matching REGEX
#   tools/gpu.sh sanitize TAG                compute-sanitizer racecheck / synccheck / memcheck on the toy smoke
set -u
mkdir -p gpurun_out
cmd=$1; shift
case "$cmd" in
  tests)
    if [ $# -gt 0 ]; then timeout 1700 python -m pytest tests -m gpu -x -q -k "$1" 2>&1 | tail -15
    else timeout 1700 python -m pytest tests -m gpu -x -q --durations=15 2>&1 | tail -25; fi ;;
  bench)
    TAG=$1; shift
    timeout 1200 python bench.py "$@" > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
    tail -c 600 gpurun_out/bench_${TAG}.json; tail -3 gpurun_out/bench_${TAG}.err ;;
  launches)
    bash tools/launch_list.sh "$1" ;;
  ncu)
    TAG=$1; RE=$2; SKIP=${3:-1}; CNT=${4:-1}
    timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${RE}" --launch-skip ${SKIP} \
      --launch-count ${CNT} -o gpurun_out/prof_${TAG} -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
      --no-e2e > gpurun_out/ncu_${TAG}.log 2>&1
    tail -3 gpurun_out/ncu_${TAG}.log ;;
  sanitize)
    TAG=$1
    for tool in memcheck racecheck synccheck; do
      timeout 1500 compute-sanitizer --tool ${tool} --print-limit 20 --target-processes all python \
        tools/sanitize_target.py > gpurun_out/sanitize_${tool}_${TAG}.log 2>&1
      echo "${tool}: rc=$?"; tail -4 gpurun_out/sanitize_${tool}_${TAG}.log
    done ;;
  *) echo "unknown: $cmd"; exit 2 ;;
esac
