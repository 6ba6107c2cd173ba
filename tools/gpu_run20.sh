# B > g in the ct-ct plans: step-3 rotations by multiples of n are the identity (lift)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "qk_ct_ct or softmax" 2>&1 | tail -3
bash tools/exp_ab.sh BLB_BSGS "qk:32" bsgsqk
