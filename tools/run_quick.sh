#!/bin/bash
# GPU test suite + quick kernel timings of cfg1..cfg5 (no e2e / CPU baseline)
TAG=${1:-q}
export PDG_JIT_CACHE=/tmp/pdg_jit
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests_${TAG}.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/tests_${TAG}.log
for c in ${CONFIGS:-cfg4 cfg2 cfg3 cfg1 cfg5}; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/q_${c}_${TAG}.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/q_${c}_${TAG}.json')); print('$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()}, 'frac', round(d['roofline']['frac'],3))"
done
