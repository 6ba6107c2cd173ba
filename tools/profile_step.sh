#!/bin/bash
# One-GPU profiling pass (run under gpurun from the repo root):
#   1. ncu launch list of one timed bench step (NVTX range "timed_steps"), serialised, cold-cache
#   2. standalone NTT throughput
#   3. ncu --set full of the top kernels (forward N=2^16 NTT passes in a 960-row batch, k_mac_tma)
# Outputs land in gpurun_out/ with the given tag.
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 900 ncu --nvtx --nvtx-include "timed_steps/" --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_bench_${TAG}.log 2>&1
timeout 300 python tools/bench_ntt.py > gpurun_out/ntt_${TAG}.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ntt16_pass --launch-skip 8 --launch-count 2 \
  -o gpurun_out/prof_ntt_${TAG} -f python tools/bench_ntt.py --rows 960 --iters 2 > gpurun_out/ncu_ntt_${TAG}.log 2>&1
