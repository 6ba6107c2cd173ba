# weight-MAC ring depth / CTAs per SM variants (STG stages, MINB CTAs/SM) on the AccG kernel
bash tools/exp_ab.sh BLB_SO "paper_2508_19525_b200/libblb.so paper_2508_19525_b200/libblb_m33.so paper_2508_19525_b200/libblb_m62.so paper_2508_19525_b200/libblb_m34.so" mstg
