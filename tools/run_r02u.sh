#!/bin/bash
mkdir -p gpurun_out
export PDG_JIT_CACHE=/tmp/pdg_jit
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/tests_r02u.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/tests_r02u.log
TREES=". ab_base" N=400000 CFG=cfg5 bash tools/ab_multi.sh
TREES=". ab_base" N=100000 CFG=cfg2 bash tools/ab_multi.sh
TREES=". ab_base" N=250000 CFG=cfg3p2 bash tools/ab_multi.sh
TREES=". ab_base" N=250000 CFG=cfg3p3 bash tools/ab_multi.sh
TREES=". ab_base" N=250000 CFG=cfg3 bash tools/ab_multi.sh
