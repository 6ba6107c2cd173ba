# P c folded into the key-switch accumulators: parity (all accumulator variants) + A/B against the previous build
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bert.py -x -q 2>&1 | tail -2
bash tools/exp_ab.sh BLB_SO "paper_2508_19525_b200/libblb_prev.so paper_2508_19525_b200/libblb.so paper_2508_19525_b200/libblb_prev.so paper_2508_19525_b200/libblb.so" pcfold
