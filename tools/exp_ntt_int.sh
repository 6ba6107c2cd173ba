mkdir -p gpurun_out
for lib in libblb.so libblb_ntt3.so; do
  echo "$lib p0: $(timeout 120 python tools/bench_ntt.py --lib paper_2508_19525_b200/$lib --prime 0 --rows 60,240,960 2>&1 | tail -1)"
done > gpurun_out/exp1.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ntt16_int --launch-skip 6 --launch-count 2 \
  -o gpurun_out/prof_ntt_int -f python tools/bench_ntt.py --prime 0 --rows 960 --iters 2 > gpurun_out/ncu_ntt_int.log 2>&1
cat gpurun_out/exp1.log
