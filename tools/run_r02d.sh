#!/bin/bash
# quick parity subset + A/B (current tree vs ab_base) on cfg5 / cfg2 / cfg4 shaped meshes
TAG=${1:-r02d}
mkdir -p gpurun_out
export PDG_JIT_CACHE=/tmp/pdg_jit
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_unit_kernels.py tests/test_oracle_golden.py tests/test_distributed_device.py -m gpu -q -x > gpurun_out/tests_${TAG}.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/tests_${TAG}.log
N=400000 CFG=cfg5 bash tools/ab_run.sh
EXTRA="PDG_ELEM_HDR=0" N=400000 CFG=cfg5 STEPS=10 bash -c 'cd . && for rep in 1 2; do env PDG_ELEM_HDR=0 PDG_JIT_CACHE=/tmp/pdg_jit timeout 600 python bench.py --config cfg5 --n 400000 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ab.json 2>/tmp/ab.err; echo "[hdr=0] rep$rep $(python -c "import json; d=json.load(open(\"/tmp/ab.json\")); print(round(d[\"phases_ms\"][\"element_kernel\"],3), \"ms el-kernel\")")"; done'
N=100000 CFG=cfg2 bash tools/ab_run.sh
N=56 CFG=cfg4 bash tools/ab_run.sh
