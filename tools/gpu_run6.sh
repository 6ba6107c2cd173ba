# BSGS retune after AccG + two-stream NTT (one MatMul varied at a time)
bash tools/exp_ab.sh BLB_BSGS "qkv:64 qkv:32 qkv:128 ffn1:32 ffn1:128 ffn2:8 ffn2:32 oproj:8 oproj:32" bsgs
