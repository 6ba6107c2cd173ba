#!/bin/bash
# MAC kernel variants on the QKV plan (BLB_MAC_TMA: 1 = 2-output grouped, 4 = 4-output grouped, 2 = single-output)
for v in 1 4 2; do
  echo "variant $v: $(BLB_MAC_TMA=$v timeout 200 python tools/bench_mac.py --plan qkv 2>&1 | tail -1)"
  echo "variant $v ffn2: $(BLB_MAC_TMA=$v timeout 200 python tools/bench_mac.py --plan ffn2 2>&1 | tail -1)"
done
