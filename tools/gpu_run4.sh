# Acc60 (60-bit rows of the key-switch inner product) parity + A/B
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "accumulator_variants or keyswitch or rotation or qk" 2>&1 | tail -2
BLB_KS_ACC=3 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "matmul or bert_size" 2>&1 | tail -2
bash tools/exp_ab.sh BLB_KS_ACC "1 3" ksacc60
