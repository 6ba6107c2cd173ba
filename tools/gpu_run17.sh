# driver-style checks: smoke() and the default bench line with its wall time
( time timeout 900 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" ) 2>&1 | tail -5
( time timeout 900 python bench.py > gpurun_out/bench_default.json ) 2>&1 | tail -4
python -c "import json; d=json.load(open('gpurun_out/bench_default.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
