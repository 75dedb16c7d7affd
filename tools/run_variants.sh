#!/bin/bash
# GPU tests + element-kernel variants on a 400k-element cfg5-shaped mesh
export PDG_JIT_CACHE=/tmp/pdg_jit
python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/tests.log 2>&1
tail -2 gpurun_out/tests.log
for v in ${VARIANTS:-"PDG_JIT_MINBLOCKS=4" "PDG_JIT_MINBLOCKS=3"}; do
  env $v python bench.py --n ${N:-400000} --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/var.json 2> gpurun_out/var.err
  echo "$v $(python -c "import json,sys; d=json.load(open('gpurun_out/var.json')); print(round(d['phases_ms']['element_kernel'],2), 'ms', round(d['roofline']['frac'],3))" 2>&1 | tail -1)"
done
