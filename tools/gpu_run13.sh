# shared-digit key-switch chunks with tighter launch bounds (3 / 4 CTAs per SM)
BLB_KS_SG=8 bash tools/exp_ab.sh BLB_SO "paper_2508_19525_b200/libblb.so paper_2508_19525_b200/libblb_sg3.so paper_2508_19525_b200/libblb_sg4.so" sgminb
bash tools/exp_ab.sh BLB_KS_SG "0" sgoff
