# round-end: all GPU tests, smoke, default bench line, ncu launch list of one step
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_r1end4.json 2> gpurun_out/bench_r1end4.err
python -c "import json; d=json.load(open('gpurun_out/bench_r1end4.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['ntt']['limbs_per_s'], d['clocks'])"
timeout 600 python bench.py --dims large --no-cpu-baseline > gpurun_out/bench_large4.json 2> gpurun_out/bench_large4.err
python -c "import json; d=json.load(open('gpurun_out/bench_large4.json')); print('large', d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
bash tools/launch_list.sh r1end4 > /dev/null 2>&1; head -12 gpurun_out/launch_shares_r1end4.md
