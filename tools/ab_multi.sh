#!/bin/bash
# on the GPU box: alternate several source trees (TREES=". ab_base ab_v1 ...") on the same mesh
export PDG_JIT_CACHE=/tmp/pdg_jit
mkdir -p gpurun_out
N=${N:-400000}; CFG=${CFG:-cfg5}; TREES=${TREES:-". ab_base"}
python bench.py --config $CFG --n $N --steps 1 --warmup 1 --profile > /dev/null 2>&1
for rep in 1 2 3; do
  for tree in $TREES; do
    (cd $tree && env $EXTRA timeout 600 python bench.py --config $CFG --n $N --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline \
       > /tmp/ab.json 2> /tmp/ab.err)
    echo "$CFG [$tree] rep$rep $(python -c "import json; d=json.load(open('/tmp/ab.json')); print(round(d['phases_ms']['element_kernel'],3), 'ms el-kernel', round(d['phases_ms']['prepass'],3), 'ms prepass', round(d['roofline']['frac'],4), 'frac')" 2>&1 | tail -1)"
  done
done
