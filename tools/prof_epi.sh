#!/bin/bash
# ncu --set full of the ModDown-epilogue NTT pass (FP64 and integer kernels) and the plain last pass
# inside one QKV ct-pt MatMul (N = 2^16)
TAG=${1:-s6}
mkdir -p gpurun_out
for K in "f64 0 0 0 1" "int 0 0 0 1" "f64 0 0 0 0"; do
  set -- $K
  F=ntt16_$1$2$3$4$5
  R="ntt16_$1<\\(bool\\)$2, \\(bool\\)$3, \\(int\\)$4, \\(int\\)$5>"
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$R" --launch-skip 1 --launch-count 1 \
    -o gpurun_out/prof_${F}_${TAG} -f python tools/bench_mac.py --plan qkv --iters 1 > gpurun_out/ncu_${F}_${TAG}.log 2>&1
done
ls gpurun_out
