# NTT occupancy variants beside the two-stream schedule: integer kernel at 3 CTAs/SM (80 registers),
# FP64 kernel at 2 CTAs/SM
bash tools/exp_ab.sh BLB_SO "paper_2508_19525_b200/libblb.so paper_2508_19525_b200/libblb_i3.so paper_2508_19525_b200/libblb_f2.so paper_2508_19525_b200/libblb_i3f2.so" so
