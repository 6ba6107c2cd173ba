#!/bin/bash
# Same-box A/B of compile-time kernel variants: each paper_2508_19525_b200/libblb_<v>.so (built with
# _build.build(defines=..., out=...)) is swapped in for libblb.so and timed with the default bench step.
#   tools/ab_so.sh TAG base v1 v2 ...     (base = the current libblb.so)
TAG=$1; shift
mkdir -p gpurun_out
cp paper_2508_19525_b200/libblb.so paper_2508_19525_b200/libblb_base.so
for rep in 1 2; do
  for v in "$@"; do
    cp paper_2508_19525_b200/libblb_${v}.so paper_2508_19525_b200/libblb.so
    touch paper_2508_19525_b200/libblb.so
    timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-f2 > gpurun_out/ab_${TAG}_${v}_${rep}.json 2>/dev/null
    python - "$v" "gpurun_out/ab_${TAG}_${v}_${rep}.json" <<'PY'
import json, sys
d = json.load(open(sys.argv[2]))
r = d["roofline"]
print("%-10s %8.3f ms  mac %.2f ms (%.0f GB/s)  ntt %.2f ms  ks %.3f" % (sys.argv[1], d["value"], r["ms_per_launch"] * 4,
      r["achieved"], d["ntt"]["share_of_step"] * d["value"], d["ks_inner"]["share_of_step"] * d["value"]))
PY
  done
done
cp paper_2508_19525_b200/libblb_base.so paper_2508_19525_b200/libblb.so
