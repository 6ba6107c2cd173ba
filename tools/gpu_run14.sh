# limb-interleaved grids (BLB_MIX: 60-bit and 40-bit limb CTAs in flight together) in the weight MAC,
# mask MAC and key-switch inner product
bash tools/exp_ab.sh BLB_SO "paper_2508_19525_b200/libblb.so paper_2508_19525_b200/libblb_mix.so paper_2508_19525_b200/libblb.so paper_2508_19525_b200/libblb_mix.so" mix
BLB_KS_SG=8 bash tools/exp_ab.sh BLB_SO "paper_2508_19525_b200/libblb_sg4.so" sg4b
