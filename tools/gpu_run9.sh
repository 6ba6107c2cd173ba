# e2e with separate upload / download streams; ncu --set full of the mask MAC (k_mac_j)
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_e2e2.json 2> gpurun_out/bench_e2e2.err
python -c "import json; d=json.load(open('gpurun_out/bench_e2e2.json')); print('value', d['value'], 'e2e', d['e2e'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mac_j --launch-skip 1 --launch-count 1 \
  -o gpurun_out/prof_macj -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_macj.log 2>&1
