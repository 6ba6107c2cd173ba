# parity (all GPU tests) with the AccG defaults, the full bench line, tensor-sum A/B, ncu of the weight MAC
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -c 600 gpurun_out/bench_full.json
bash tools/exp_ab.sh BLB_TSUM_ACC "0 1" tsum
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mac_tma4 --launch-count 1 \
  -o gpurun_out/prof_mac_g2 -f python tools/bench_mac.py --plan qkv --iters 1 > gpurun_out/ncu_mac_g2.log 2>&1
