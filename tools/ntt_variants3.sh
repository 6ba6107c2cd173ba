#!/bin/bash
for lib in libblb.so libblb_p3.so; do
  echo "$lib prime 1: $(timeout 120 python tools/bench_ntt.py --lib paper_2508_19525_b200/$lib --prime 1 --rows 300,960 2>&1 | tail -1)"
  echo "$lib mixed: $(timeout 120 python tools/bench_ntt.py --lib paper_2508_19525_b200/$lib --rows 300,960 2>&1 | tail -1)"
done
