#!/bin/bash
# one full ncu capture of the element kernel (1 GPU, short run)
CFG=${1:-cfg5}; N=${2:-100000}; TAG=${3:-v0}
ncu --set full --clock-control none --import-source on -k regex:assemble_elements -s 1 -c 1 \
    -o gpurun_out/prof_${CFG}_${TAG} python bench.py --config $CFG --n $N --steps 1 --warmup 1 --profile \
    > gpurun_out/ncu_${CFG}_${TAG}.log 2>&1
