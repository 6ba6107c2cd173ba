timeout 200 python tools/bench_ntt.py --prime 1 --rows 960 > gpurun_out/ntt_p1.json 2>&1; cat gpurun_out/ntt_p1.json
timeout 200 python tools/bench_ntt.py --prime 0 --rows 960 > gpurun_out/ntt_p0.json 2>&1; cat gpurun_out/ntt_p0.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ntt16_pass --launch-skip 6 --launch-count 2 -o gpurun_out/prof_ntt_f64 -f python tools/bench_ntt.py --prime 1 --rows 960 --iters 2 > gpurun_out/ncu_ntt_f64.log 2>&1
bash tools/profile_kernels.sh f64
ls gpurun_out/
