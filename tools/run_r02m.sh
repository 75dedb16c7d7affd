#!/bin/bash
TAG=${1:-r02m}
mkdir -p gpurun_out
export PDG_JIT_CACHE=/tmp/pdg_jit
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_oracle_golden.py -m gpu -q -x > gpurun_out/tests_${TAG}.log 2>&1
echo "parity rc=$?"; tail -1 gpurun_out/tests_${TAG}.log
PDG_JIT_DEFINES="-DPDG_COLS_PER_IFACE=1" timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_oracle_golden.py -m gpu -q -x > gpurun_out/tests_cpi_${TAG}.log 2>&1
echo "parity cols-per-iface rc=$?"; tail -1 gpurun_out/tests_cpi_${TAG}.log
python bench.py --n 400000 --steps 1 --warmup 1 --profile > /dev/null 2>&1
PDG_JIT_DEFINES="-DPDG_TIMERS=1" timeout 600 python bench.py --n 400000 --steps 2 --warmup 1 --profile 2>&1 | grep PDG_TIMERS | head -2
for rep in 1 2 3; do
  for v in base cpi abb; do
    if [ $v = abb ]; then d=ab_base; def=""; else d=.; def=""; [ $v = cpi ] && def="-DPDG_COLS_PER_IFACE=1"; fi
    (cd $d && PDG_JIT_DEFINES="$def" timeout 600 python bench.py --n 400000 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ab.json 2>/tmp/ab.err)
    echo "cfg5 [$v] rep$rep $(python -c "import json; d=json.load(open('/tmp/ab.json')); print(round(d['phases_ms']['element_kernel'],3))")"
  done
done
