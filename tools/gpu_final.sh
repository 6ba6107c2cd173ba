# Round-end evidence: full bench line, ncu launch list of one step, ncu --set full of the mask MAC
# (k_mac_j) and the key-switch inner product; run from the repo root under gpurun
TAG=${1:-final}
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
tail -c 400 gpurun_out/bench_${TAG}.json
bash tools/launch_list.sh ${TAG}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mac_j --launch-skip 1 --launch-count 1 \
  -o gpurun_out/prof_macj_${TAG} -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_macj_${TAG}.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ntt16 --launch-skip 40 --launch-count 4 \
  -o gpurun_out/prof_ntt_${TAG} -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_ntt_${TAG}.log 2>&1
ls gpurun_out | grep ${TAG}
