#!/bin/bash
# Round-2 (second session) evidence on the final code: GPU suite, default bench line, BERT-large, GPT2
# config 5, per-block times, launch list of one step, ncu --set full of the top kernels.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/r2s2_gpu_tests.log 2>&1; tail -3 gpurun_out/r2s2_gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2s2_bench.json 2> gpurun_out/r2s2_bench.err
tail -c 300 gpurun_out/r2s2_bench.json; echo
timeout 900 python bench.py --dims large --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2s2_bench_large.json 2> gpurun_out/r2s2_bench_large.err
timeout 900 python bench.py --model gpt2 --steps 2 --warmup 1 > gpurun_out/r2s2_bench_gpt2_config5.json 2> gpurun_out/r2s2_bench_gpt2.err
python tools/block_times.py --steps 5 --warmup 2 > gpurun_out/r2s2_block_times.json 2>&1; cat gpurun_out/r2s2_block_times.json
bash tools/launch_list.sh r2s2 > /dev/null 2>&1; head -12 gpurun_out/launch_shares_r2s2.md
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mac_tma4|k_ks_bulk|k_mac_j" --launch-count 6 \
  -o gpurun_out/prof_r2s2_top -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-f2 > gpurun_out/ncu_r2s2_top.log 2>&1
tail -1 gpurun_out/ncu_r2s2_top.log
