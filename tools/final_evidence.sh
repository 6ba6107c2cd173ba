#!/bin/bash
# Round-end evidence on one B200 (run from the repo root under gpurun):
#   -m gpu suite, smoke, the default bench line, BERT-large, the config-5 stack, a 2-rank functional
#   run, the ncu launch list of one timed step, and ncu --set full of the top kernels.
TAG=${1:-r2final}
mkdir -p gpurun_out
timeout 1700 python -m pytest tests -m gpu -x -q --durations=12 > gpurun_out/tests_${TAG}.log 2>&1; tail -3 gpurun_out/tests_${TAG}.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}.json')); print('base', d['value'], d['e2e']['value'], d['roofline']['frac'], d['ntt']['limbs_per_s'], d['full_layer']['ms'], d['clocks'])"
timeout 900 python bench.py --dims large --steps 10 --warmup 3 --no-cpu-baseline --no-f2 > gpurun_out/bench_large_${TAG}.json 2> gpurun_out/bench_large_${TAG}.err
python -c "import json; d=json.load(open('gpurun_out/bench_large_${TAG}.json')); print('large', d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 1 --no-cpu-baseline --no-f2 --no-e2e > gpurun_out/bench_2rank_${TAG}.json 2> gpurun_out/bench_2rank_${TAG}.err
tail -c 300 gpurun_out/bench_2rank_${TAG}.json; tail -2 gpurun_out/bench_2rank_${TAG}.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
tail -c 300 gpurun_out/bench_ref_${TAG}.json
bash tools/launch_list.sh ${TAG} > /dev/null 2>&1; head -24 gpurun_out/launch_shares_${TAG}.md
bash tools/gpu.sh ncu mac_${TAG} k_mac_tma4 0 1
bash tools/gpu.sh ncu ks_${TAG} k_ks_inner 8 2
bash tools/gpu.sh ncu ntt_${TAG} ntt16 40 4
bash tools/gpu.sh ncu macj_${TAG} k_mac_j 0 1
ls gpurun_out | grep ${TAG}
