#!/bin/bash
# copy one evidence session's outputs (tools/run_evidence.sh TAG) into profiles/ as <NAME>
TAG=$1; NAME=${2:-$1}
set -e
for f in gpurun_out/bench_*_${TAG}.json gpurun_out/bench[248]_*_${TAG}.json; do
  b=$(basename $f .json); b=${b%_${TAG}}
  cp $f profiles/${b}_${NAME}.json
done
cp gpurun_out/launches_cfg5_${TAG}.csv profiles/launches_cfg5_${NAME}.csv
for r in gpurun_out/prof_*_${TAG}.ncu-rep; do
  c=$(basename $r .ncu-rep); c=${c#prof_}; c=${c%_${TAG}}
  python tools/ncu_summary.py $r 40 > profiles/ncu_${c}_${NAME}.txt 2>&1 || true
done
cp gpurun_out/tests_${TAG}.log profiles/tests_gpu_${NAME}.log 2>/dev/null || true
cp gpurun_out/smoke_${TAG}.log profiles/smoke_${NAME}.log 2>/dev/null || true
cp gpurun_out/box_${TAG}.txt profiles/box_${NAME}.txt 2>/dev/null || true
for t in memcheck racecheck synccheck initcheck; do
  [ -f gpurun_out/sanitizer_${t}_${TAG}.log ] && grep -vE "^=========     (Host Frame|Saved host)" gpurun_out/sanitizer_${t}_${TAG}.log | head -400 > profiles/sanitizer_${t}_${NAME}.log
done
python tools/traffic_json.py ${NAME}
echo collected
