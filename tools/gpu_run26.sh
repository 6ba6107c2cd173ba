# prologue reduction skip via per-launch digit masks (no per-row prime lookup): parity + A/B vs the previous build
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "matmul or keyswitch or rotation or qk or bert" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_bert.py -x -q 2>&1 | tail -2
bash tools/exp_ab.sh BLB_SO "paper_2508_19525_b200/libblb_prev.so paper_2508_19525_b200/libblb.so paper_2508_19525_b200/libblb_prev.so paper_2508_19525_b200/libblb.so" prored2
