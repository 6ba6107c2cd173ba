#!/bin/bash
# Round-2 (second session) evidence on the final code: default bench line, BERT-large, per-block times,
# launch list of one step, ncu --set full of the top kernels.
set -u
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2s2_bench.json 2> gpurun_out/r2s2_bench.err
tail -c 400 gpurun_out/r2s2_bench.json; echo
timeout 900 python bench.py --dims large --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2s2_bench_large.json 2> gpurun_out/r2s2_bench_large.err
python tools/block_times.py --steps 5 --warmup 2 > gpurun_out/r2s2_block_times.json 2>&1; cat gpurun_out/r2s2_block_times.json
bash tools/launch_list.sh r2s2 > /dev/null 2>&1; head -12 gpurun_out/launch_shares_r2s2.md
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mac_tma4|k_ks_bulk|k_mac_j" --launch-count 6 \
  -o gpurun_out/prof_r2s2_top -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-f2 > gpurun_out/ncu_r2s2_top.log 2>&1
tail -1 gpurun_out/ncu_r2s2_top.log
