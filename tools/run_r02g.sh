#!/bin/bash
# bulk-copy (TMA) A/B, parity with the bulk variant, compute-sanitizer logs
TAG=${1:-r02g}
mkdir -p gpurun_out
export PDG_JIT_CACHE=/tmp/pdg_jit
PDG_JIT_DEFINES="-DPDG_BULK=1" timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_oracle_golden.py -m gpu -q -x > gpurun_out/tests_bulk_${TAG}.log 2>&1
echo "bulk parity rc=$?"; tail -1 gpurun_out/tests_bulk_${TAG}.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_unit_kernels.py tests/test_oracle_golden.py -m gpu -q -x > gpurun_out/tests_${TAG}.log 2>&1
echo "parity rc=$?"; tail -1 gpurun_out/tests_${TAG}.log
TREES=". ab_base" N=400000 CFG=cfg5 bash tools/ab_multi.sh
for rep in 1 2 3; do (PDG_JIT_DEFINES="-DPDG_BULK=1" timeout 600 python bench.py --config cfg5 --n 400000 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ab.json 2>/tmp/ab.err; echo "cfg5 [bulk] rep$rep $(python -c "import json; d=json.load(open('/tmp/ab.json')); print(round(d['phases_ms']['element_kernel'],3), 'ms el-kernel')")"); done
TREES=". ab_base" N=100000 CFG=cfg2 bash tools/ab_multi.sh
TREES=". ab_base" N=56 CFG=cfg4 bash tools/ab_multi.sh
# compute-sanitizer on small golden cases (cfg1-size Voronoi p=1, 3D ADR, advdiff3d)
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python -m pytest tests/test_oracle_golden.py -m gpu -q \
     -k "engine and (cfg1_voronoi1000 or cube3_adr or cube4_advdiff3d or voronoi120_poisson_p4)" \
     > gpurun_out/sanitizer_${tool}_${TAG}.log 2>&1
  echo "sanitizer $tool rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitizer_${tool}_${TAG}.log | tail -2 | tr '\n' ' ')"
done
