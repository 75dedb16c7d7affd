#!/bin/bash
# ncu full capture of the element kernel on a 100k cfg5-shaped mesh (tag $1)
export PDG_JIT_CACHE=/tmp/pdg_jit
python bench.py --n 100000 --steps 1 --warmup 1 --profile > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pdg_jit_kernel -s 1 -c 1 \
    -o gpurun_out/prof_cfg5_$1 python bench.py --n 100000 --steps 1 --warmup 1 --profile > gpurun_out/ncu_$1.log 2>&1
