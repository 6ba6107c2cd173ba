# ct-ct BSGS baby-step count B (g | B | L; default g = 16) for Q K^T and Softmax x V
bash tools/exp_ab.sh BLB_BSGS "qk:16 qk:32 qk:64" bsgsqk
