#!/bin/bash
export PDG_JIT_CACHE=/tmp/pdg_jit
python bench.py --n 400000 --steps 1 --warmup 1 --profile > /dev/null 2>&1
for d in "" "-DPDG_VOL_UNROLL=2" "-DPDG_FACE_UNROLL=2" "-DPDG_VOL_UNROLL=2 -DPDG_FACE_UNROLL=2" "-DPDG_RULES_SMEM=0"; do
  r=$(PDG_JIT_DEFINES="$d" timeout 600 python bench.py --n 400000 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['phases_ms']['element_kernel'],3))")
  echo "defines=[$d] element_ms=$r"
done
