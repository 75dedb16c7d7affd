#!/bin/bash
# full GPU tests, cfg2 bench (with the assemble_approach2 e2e leg), ncu --set full captures of the element kernel
TAG=${1:-r02j}
mkdir -p gpurun_out
export PDG_JIT_CACHE=/tmp/pdg_jit
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/tests_${TAG}.log 2>&1
echo "tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/tests_${TAG}.log | tail -6
timeout 900 python bench.py --config cfg2 --steps 5 --warmup 3 > gpurun_out/bench_cfg2_${TAG}.json 2> gpurun_out/bench_cfg2_${TAG}.err
echo "bench cfg2 rc=$?"; python -c "import json; d=json.load(open('gpurun_out/bench_cfg2_${TAG}.json')); print(d['value'], d['ms_per_step'], d.get('e2e'), d.get('e2e_api'))"
for c in "cfg5 400000" "cfg2 100000" "cfg3 250000" "cfg4 56" "cfg3p3 250000"; do
  set -- $c
  python bench.py --config $1 --n $2 --steps 1 --warmup 1 --profile > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:pdg_jit_kernel -s 1 -c 1 \
      -o gpurun_out/prof_${1}_${TAG} python bench.py --config $1 --n $2 --steps 1 --warmup 1 --profile \
      > gpurun_out/ncu_${1}_${TAG}.log 2>&1
  echo "ncu $1 rc=$?"
done
