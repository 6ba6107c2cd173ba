#!/bin/bash
# NTT occupancy variants: default (2 CTAs/SM), BLB_NTT_MINB=3, =4, per prime size
for lib in libblb.so libblb_ntt3.so libblb_ntt4.so; do
  for p in 1 0; do
    echo "$lib prime $p: $(timeout 120 python tools/bench_ntt.py --lib paper_2508_19525_b200/$lib --prime $p --rows 960 2>&1 | tail -1)"
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ks_inner --launch-skip 3 --launch-count 1 \
  -o gpurun_out/prof_ksinner -f python tools/bench_mac.py --plan qkv --iters 1 > gpurun_out/ncu_ksinner.log 2>&1
