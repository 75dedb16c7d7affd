#!/bin/bash
# warps-per-CTA variants of the slab kernel on reduced slab workloads
export PDG_JIT_CACHE=/tmp/pdg_jit
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_slab_oracle.py -m gpu -x -q 2>&1 | tail -2
for c in st1 st2 st3 st4; do
  for w in default 1 2 4; do
    if [ $w = default ]; then unset PDG_SLAB_WARPS; else export PDG_SLAB_WARPS=$w; fi
    r=$(timeout 300 python bench.py --config $c --n 200000 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['phases_ms']['element_kernel'],2), round(d['roofline']['frac'],3))")
    echo "$c warps=$w element_ms frac: $r"
  done
done
