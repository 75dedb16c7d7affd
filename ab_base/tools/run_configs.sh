#!/bin/bash
# bench lines for every BASELINE.json config on one GPU (cfg3 as its p = 2..6 sweep)
TAG=${1:-r01}
export PDG_JIT_CACHE=/tmp/pdg_jit
mkdir -p gpurun_out
run() {  # name, args...
  local name=$1; shift
  timeout 1500 python bench.py "$@" > gpurun_out/bench_${name}_${TAG}.json 2> gpurun_out/bench_${name}_${TAG}.err
  echo "$name rc=$? $(python -c "import json,sys; d=json.load(open('gpurun_out/bench_${name}_${TAG}.json')); print(round(d['value']/1e6,3),'M el/s', round(d['ms_per_step'],3),'ms', 'frac', round(d['roofline']['frac'],3), 'e2e', round(d.get('e2e',{}).get('value',0)/1e6,3), 'cpu', round(d.get('cpu_baseline',{}).get('value',0),1))" 2>&1 | tail -1)"
}
run cfg1 --config cfg1 --steps 20 --warmup 5
run cfg2 --config cfg2
for p in 2 3 4 5 6; do run cfg3p$p --config cfg3 --degree $p; done
run cfg4 --config cfg4
