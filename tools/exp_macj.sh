#!/bin/bash
# A/B of the mask-MAC variants (BLB_MAC_J = 0: per-output k_mac, 2 / 4: k_mac_j groups)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "qk or softmax" > gpurun_out/macj_tests.log 2>&1; echo "rc=$?" >> gpurun_out/macj_tests.log
BLB_MAC_J=4 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "qk or softmax" >> gpurun_out/macj_tests.log 2>&1; echo "rc4=$?" >> gpurun_out/macj_tests.log
for v in 0 2 4; do
  BLB_MAC_J=$v timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_macj$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bench_macj$v.json')); print('MAC_J=$v', d['value'], d['mask_mac'])"
done
tail -4 gpurun_out/macj_tests.log
