#!/bin/bash
# ncu --set full captures of the top kernels of one ct-pt MatMul (QKV plan, N = 2^16):
# the TMA MAC, the ModDown-epilogue NTT pass and the ModUp-prologue NTT pass.
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mac_tma4 --launch-count 1 \
  -o gpurun_out/prof_mactma_${TAG} -f python tools/bench_mac.py --plan qkv --iters 1 > gpurun_out/ncu_mactma_${TAG}.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:ntt16_pass<0, 0, 0, 1>" --launch-skip 2 --launch-count 1 \
  -o gpurun_out/prof_ntt_epi_${TAG} -f python tools/bench_mac.py --plan qkv --iters 1 > gpurun_out/ncu_ntt_epi_${TAG}.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:ntt16_pass<0, 1, 1, 0>" --launch-skip 2 --launch-count 1 \
  -o gpurun_out/prof_ntt_pro_${TAG} -f python tools/bench_mac.py --plan qkv --iters 1 > gpurun_out/ncu_ntt_pro_${TAG}.log 2>&1
