# two-stream NTT (integer rows on the auxiliary stream): parity + A/B
BLB_NTT_2S=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layer.py -x -q 2>&1 | tail -2
bash tools/exp_ab.sh BLB_NTT_2S "0 1" ntt2s
