#!/bin/bash
export PDG_JIT_CACHE=/tmp/pdg_jit
python bench.py --n 400000 --steps 1 --warmup 1 --profile > /dev/null 2>&1
for v in "4 3" "2 6" "1 12" "2 5" "4 2"; do
  set -- $v
  r=$(PDG_JIT_WARPS=$1 PDG_JIT_MINBLOCKS=$2 timeout 600 python bench.py --n 400000 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['phases_ms']['element_kernel'],3))")
  echo "warps=$1 minblocks=$2 element_ms=$r"
done
