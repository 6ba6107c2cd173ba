#!/bin/bash
# weight-MAC variants: plaintext packing (BLB_PT_PACK) x c0 products on FP64 (BLB_MAC_F64)
mkdir -p gpurun_out
for pk in 0 1; do for f in 0 1; do
  BLB_PT_PACK=$pk BLB_MAC_F64=$f timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_pk${pk}_f${f}.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_pk${pk}_f${f}.json'))
print('pack=$pk f64=$f', round(d['value'],2), 'mac', round(d['roofline']['share_of_step']*d['value'],2), round(d['roofline']['achieved']), 'GB/s')"
done; done
BLB_MAC_F64=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "matmul or toy" 2>&1 | tail -1
BLB_PT_PACK=0 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "matmul or toy" 2>&1 | tail -1
