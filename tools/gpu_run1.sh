set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
BLB_MAC_NINT=-1 timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash tools/exp_ab.sh BLB_MAC_NINT "0 -1" macg
