#!/bin/bash
# key-switch batch size for independent rotations (L2 residency of the extended digits)
for b in 32 16 8 6 4; do
  echo "batch $b: $(BLB_INDEP_BATCH=$b timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ks_inner"], d["ntt"]["share_of_step"])')"
done
