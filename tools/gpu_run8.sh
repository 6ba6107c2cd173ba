# key-switch 60-bit rows one job at a time on Acc60 (BLB_KS_ACC=4): parity + A/B; integer NTT at 3 CTAs/SM now default
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "accumulator_variants" 2>&1 | tail -2
BLB_KS_ACC=4 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layer.py -x -q 2>&1 | tail -2
bash tools/exp_ab.sh BLB_KS_ACC "1 4" ks4
