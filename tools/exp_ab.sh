#!/bin/bash
# A/B of one env knob on the bench step: tools/exp_ab.sh VAR "v1 v2 ..." [tag]
VAR=$1; VALS=$2; TAG=${3:-ab}
mkdir -p gpurun_out
for v in $VALS; do
  f="gpurun_out/bench_${TAG}_$(echo "$v" | tr '/:' '__').json"
  env $VAR=$v timeout 300 python bench.py --no-cpu-baseline --no-e2e > "$f" 2>/dev/null
  python -c "
import json, sys; d=json.load(open(sys.argv[1]))
print('$VAR=$v', round(d['value'],2), 'mac', round(d['roofline']['share_of_step']*d['value'],2), 'ntt', round(d['ntt']['share_of_step']*d['value'],2),
      'ks', round(d['ks_inner']['share_of_step']*d['value'],2), 'mmac', round(d['mask_mac']['share_of_step']*d['value'],2),
      'tsum', round((d.get('tensor_sum',{}).get('share_of_step') or 0)*d['value'],2))" "$f"
done
