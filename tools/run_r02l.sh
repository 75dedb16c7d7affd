#!/bin/bash
TAG=${1:-r02l}
mkdir -p gpurun_out
export PDG_JIT_CACHE=/tmp/pdg_jit
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_oracle_golden.py tests/test_unit_kernels.py tests/test_approach1.py -m gpu -q -x > gpurun_out/tests_${TAG}.log 2>&1
echo "parity rc=$?"; tail -3 gpurun_out/tests_${TAG}.log
TREES=". ab_base" N=250000 CFG=cfg3p3 bash tools/ab_multi.sh
TREES=". ab_base" N=56 CFG=cfg4 bash tools/ab_multi.sh
TREES=". ab_base" N=100000 CFG=cfg2 bash tools/ab_multi.sh
