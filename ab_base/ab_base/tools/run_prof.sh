#!/bin/bash
# GPU tests (optional) + one ncu --set full capture of the element kernel on N cells
TAG=${1:-dev}; N=${N:-400000}; CFG=${CFG:-cfg5}
export PDG_JIT_CACHE=/tmp/pdg_jit
mkdir -p gpurun_out
if [ -z "$SKIP_TESTS" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q ${TESTS:-} > gpurun_out/tests.log 2>&1
  echo "tests rc=$? $(tail -1 gpurun_out/tests.log)"
fi
python bench.py --config $CFG --n $N --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/prof_bench_${TAG}.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/prof_bench_${TAG}.json')); print('bench', d['phases_ms'], round(d['roofline']['frac'],4))"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pdg_jit_kernel -s 1 -c 1 \
    -o gpurun_out/prof_${CFG}_${TAG} python bench.py --config $CFG --n $N --steps 1 --warmup 1 --profile \
    > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu rc=$?"
