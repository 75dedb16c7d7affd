#!/bin/bash
# ncu full capture of the (NVRTC-specialised) element kernel + a cfg5 bench
export PDG_JIT_CACHE=/tmp/pdg_jit
python bench.py --n 100000 --steps 1 --warmup 1 --profile > /dev/null 2>&1   # warm the JIT cache
ncu --set full --clock-control none --import-source on -k regex:pdg_jit_kernel -s 1 -c 1 \
    -o gpurun_out/prof_cfg5_${1:-v2} python bench.py --n 100000 --steps 1 --warmup 1 --profile > gpurun_out/ncu_v2.log 2>&1
python bench.py > gpurun_out/bench_cfg5_${1:-v2}.json 2> gpurun_out/bench_cfg5_${1:-v2}.err
