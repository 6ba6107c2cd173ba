# round-end confirmation on the final code: all GPU tests, smoke, the default bench line
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_r1end.json 2> gpurun_out/bench_r1end.err
python -c "import json; d=json.load(open('gpurun_out/bench_r1end.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
