#!/bin/bash
# Full GPU test suite, the default bench line, and Approach 1 vs 2 lines.
TAG=${1:-r01}
mkdir -p gpurun_out
export PDG_JIT_CACHE=/tmp/pdg_jit
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests_${TAG}.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/tests_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_cfg5_${TAG}.json 2> gpurun_out/bench_cfg5_${TAG}.err
echo "bench cfg5 rc=$?"; head -c 700 gpurun_out/bench_cfg5_${TAG}.json; echo
for c in cfg1 cfg2 cfg3; do
  for ap in 2 1; do
    timeout 900 python bench.py --config $c --approach $ap --steps 5 --warmup 3 --no-e2e --no-cpu-baseline \
      > gpurun_out/bench_${c}_a${ap}_${TAG}.json 2> gpurun_out/bench_${c}_a${ap}_${TAG}.err
    echo "bench $c A$ap rc=$?"; python -c "import json; d=json.load(open('gpurun_out/bench_${c}_a${ap}_${TAG}.json')); print(d['ms_per_step'], d['phases_ms'])"
  done
done
