#!/bin/bash
for lib in libblb.so libblb_f64m4.so libblb_f64m2.so; do
  for p in 1 0; do
    echo "$lib prime $p: $(timeout 120 python tools/bench_ntt.py --lib paper_2508_19525_b200/$lib --prime $p --rows 960 2>&1 | tail -1)"
  done
  echo "$lib mixed: $(timeout 120 python tools/bench_ntt.py --lib paper_2508_19525_b200/$lib --rows 300,960 2>&1 | tail -1)"
done
