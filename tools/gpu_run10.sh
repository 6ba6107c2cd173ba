# shared-digit key-switch chunks (k_ks_inner_sg): parity + A/B of the chunk length
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layer.py -x -q 2>&1 | tail -2
bash tools/exp_ab.sh BLB_KS_SG "0 8 4 16" kssg
