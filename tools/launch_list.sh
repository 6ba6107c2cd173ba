#!/bin/bash
# ncu launch list of one timed bench step (NVTX range "timed_steps"), serialised, cold-cache
TAG=${1:-x}
mkdir -p gpurun_out
timeout 800 ncu --nvtx --nvtx-include "timed_steps/" --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_bench_${TAG}.log 2>&1
python tools/summarize_ncu.py --launches gpurun_out/launches_${TAG}.csv > gpurun_out/launch_shares_${TAG}.md
head -30 gpurun_out/launch_shares_${TAG}.md
