set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_layer.py tests/test_gpu_parity.py tests/test_gpu_bert.py -m gpu -x -q -k "dnum1 or layer_step or toy_config" 2>&1 | tail -5
timeout 300 python bench.py --config toy --steps 20 --warmup 3 > gpurun_out/bench_toy.json 2> gpurun_out/bench_toy.err; tail -c 1500 gpurun_out/bench_toy.json; tail -3 gpurun_out/bench_toy.err
timeout 1200 python bench.py --preset bert_dnum1 --no-f2 > gpurun_out/bench_dnum1.json 2> gpurun_out/bench_dnum1.err; tail -c 3000 gpurun_out/bench_dnum1.json; tail -3 gpurun_out/bench_dnum1.err
