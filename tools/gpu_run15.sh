# BERT-large layer (config 4 dims: hidden 1024, 16 heads, FFN 4096, L = 128) at N = 1
timeout 1200 python bench.py --dims large --no-cpu-baseline > gpurun_out/bench_large.json 2> gpurun_out/bench_large.err
tail -c 300 gpurun_out/bench_large.json; tail -3 gpurun_out/bench_large.err
