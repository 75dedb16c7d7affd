#!/bin/bash
# 3D (cfg4) element kernel: phase timers + one ncu --set full capture
export PDG_JIT_CACHE=/tmp/pdg_jit
mkdir -p gpurun_out
python bench.py --config cfg4 --steps 2 --warmup 1 --profile > gpurun_out/cfg4_bench.json 2>&1
PDG_JIT_DEFINES="-DPDG_TIMERS=1" python bench.py --config cfg4 --steps 1 --warmup 1 --profile 2>&1 | grep PDG_TIMERS | head -4 > gpurun_out/cfg4_timers.txt
ncu --set full --clock-control none --import-source on -k regex:pdg_jit_kernel -s 1 -c 1 \
    -o gpurun_out/prof_cfg4 python bench.py --config cfg4 --steps 1 --warmup 1 --profile > gpurun_out/ncu_cfg4.log 2>&1
echo "ncu rc=$?"
cat gpurun_out/cfg4_timers.txt
