# k_mac_r with 4 (default) / 16 tiles per CTA vs k_mac_j; parity of the qk tests
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "qk or softmax or accumulator" 2>&1 | tail -2
bash tools/exp_ab.sh BLB_MAC_R "0 1" macr4
bash tools/exp_ab.sh BLB_SO "paper_2508_19525_b200/libblb_t16.so" macr16
