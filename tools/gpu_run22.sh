# fused ModUp / ModDown prologue without moot reductions (BLB_PRO_RED): parity + A/B
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/exp_ab.sh BLB_PRO_RED "0 1 0 1" prored
