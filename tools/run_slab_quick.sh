#!/bin/bash
export PDG_JIT_CACHE=/tmp/pdg_jit
timeout 900 python -m pytest tests/test_slab_oracle.py -m gpu -x -q 2>&1 | tail -2
for c in ${CONFIGS:-st1 st2 st3}; do
  timeout 900 python bench.py --config $c --n ${N:-200000} --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['phases_ms']['element_kernel'],3), 'ms frac', round(d['roofline']['frac'],3))"
done
