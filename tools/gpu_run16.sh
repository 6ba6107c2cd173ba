# FP64 NTT quotient as fl(p * qinv) rounded with two adds (no uniform-register copies) vs one fma; parity of the variant
BLB_SO=paper_2508_19525_b200/libblb_rnd.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ntt or keyswitch or rotation or matmul" 2>&1 | tail -2
bash tools/exp_ab.sh BLB_SO "paper_2508_19525_b200/libblb.so paper_2508_19525_b200/libblb_rnd.so paper_2508_19525_b200/libblb.so paper_2508_19525_b200/libblb_rnd.so" rnd
