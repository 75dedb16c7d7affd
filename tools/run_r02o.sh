#!/bin/bash
mkdir -p gpurun_out
export PDG_JIT_CACHE=/tmp/pdg_jit
for t in synccheck racecheck; do compute-sanitizer --tool $t ./tools/probe/mbar_probe > gpurun_out/probe_${t}.log 2>&1; echo "probe $t: $(grep -E 'SUMMARY|Missing' gpurun_out/probe_${t}.log | sort | uniq -c | head -3)"; done
PDG_JIT_DEFINES="-DPDG_BULK=0" timeout 900 compute-sanitizer --tool synccheck python -m pytest tests/test_oracle_golden.py -m gpu -q \
  -k "engine and (cfg1_voronoi1000 or cube3_adr or cube4_advdiff3d or voronoi120_poisson_p4 or clusters6_poisson_p3)" > gpurun_out/sanitizer_synccheck_nobulk.log 2>&1
echo "synccheck nobulk: $(grep -E 'ERROR SUMMARY' gpurun_out/sanitizer_synccheck_nobulk.log | tail -1)"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_oracle_golden.py -m gpu -q -x > gpurun_out/tests_r02o.log 2>&1
echo "parity rc=$?"; tail -1 gpurun_out/tests_r02o.log
TREES=". ab_base" N=400000 CFG=cfg5 bash tools/ab_multi.sh
TREES=". ab_base" N=250000 CFG=cfg3 bash tools/ab_multi.sh
TREES=". ab_base" N=56 CFG=cfg4 bash tools/ab_multi.sh
