#!/bin/bash
# GPU tests + element-kernel variant A/B + phase timers (cfg5-shaped 400k mesh)
TAG=${1:-r02c}
mkdir -p gpurun_out
export PDG_JIT_CACHE=/tmp/pdg_jit
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/tests_${TAG}.log 2>&1
echo "tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/tests_${TAG}.log | tail -8
python bench.py --n 400000 --steps 1 --warmup 1 --profile > /dev/null 2>&1
PDG_JIT_DEFINES="-DPDG_TIMERS=1" timeout 600 python bench.py --n 400000 --steps 2 --warmup 1 --profile 2>&1 | grep PDG_TIMERS | head -4
VARIANTS=$'base\nPDG_JIT_DEFINES=-DPDG_VOL_ORDER=0\nPDG_JIT_WARPS=2|PDG_JIT_MINBLOCKS=6\nPDG_JIT_MAXNREG=200\nPDG_JIT_MAXNREG=255' SKIP_TESTS=1 bash tools/run_variants.sh
