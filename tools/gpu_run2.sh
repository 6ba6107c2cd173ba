# A/B of the grid-split FP64 accumulator (AccG) in the key-switch inner product and the mask MAC,
# parity of both, and an ncu --set full capture of the AccG weight MAC and key-switch inner product
BLB_KS_ACC=1 BLB_MACJ_ACC=2 BLB_MAC_NINT=-1 timeout 900 python -m pytest tests -m gpu -x -q -k "not bert" 2>&1 | tail -2
BLB_KS_ACC=2 BLB_MACJ_ACC=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "keyswitch or rotate or qk" 2>&1 | tail -2
bash tools/exp_ab.sh BLB_KS_ACC "1 2" ksacc
bash tools/exp_ab.sh BLB_MACJ_ACC "1 2" macjacc
BLB_MAC_NINT=-1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mac_tma4 --launch-count 1 \
  -o gpurun_out/prof_mac_g -f python tools/bench_mac.py --plan qkv --iters 1 > gpurun_out/ncu_mac_g.log 2>&1
BLB_KS_ACC=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ks_inner --launch-skip 4 --launch-count 1 \
  -o gpurun_out/prof_ks_g -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_ks_g.log 2>&1
ls -la gpurun_out
