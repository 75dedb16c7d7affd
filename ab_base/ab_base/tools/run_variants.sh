#!/bin/bash
# GPU parity tests + element-kernel variants on a cfg5-shaped mesh (N cells).
#   VARIANTS: lines of env assignments ('|' separates variables, so values may
#   contain spaces), e.g.
#   VARIANTS=$'base\nPDG_PLAIN_VOLUME=1\nPDG_JIT_DEFINES=-DPDG_VOL_SPLITC=1 -DPDG_DMMA_VOLATILE=0'
export PDG_JIT_CACHE=/tmp/pdg_jit
mkdir -p gpurun_out
if [ -z "$SKIP_TESTS" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q ${TESTS:-} > gpurun_out/tests.log 2>&1
  echo "tests rc=$? $(tail -1 gpurun_out/tests.log)"
fi
[ -n "$PRE" ] && eval "$PRE"
CFG=${CFG:-cfg5}
python bench.py --config $CFG --n ${N:-400000} --steps 1 --warmup 1 --profile > /dev/null 2>&1  # mesh cache
while IFS= read -r v; do
  [ -z "$v" ] && continue
  envs=()
  if [ "$v" != "base" ]; then IFS='|' read -ra envs <<< "$v"; fi
  for rep in 1 2; do
    env "${envs[@]}" timeout 600 python bench.py --config $CFG --n ${N:-400000} --steps ${STEPS:-10} --warmup 3 \
        --no-e2e --no-cpu-baseline > gpurun_out/var.json 2> gpurun_out/var.err
    echo "[$v] rep$rep $(python -c "import json; d=json.load(open('gpurun_out/var.json')); print(round(d['phases_ms']['element_kernel'],3), 'ms el-kernel', round(d['roofline']['frac'],4), 'frac')" 2>&1 | tail -1)"
  done
done <<< "${VARIANTS:-base}"
