#!/bin/bash
# Space-time slab session: slab parity tests, bench lines st1..st5, launch
# list of st3 and one ncu --set full capture of the slab kernel.
#   tools/gpu.sh --timeout 3000 -- 'bash tools/run_slab.sh r01'
TAG=${1:-r01}
mkdir -p gpurun_out
export PDG_JIT_CACHE=/tmp/pdg_jit
timeout 900 python -m pytest tests/test_slab_oracle.py -m gpu -x -q > gpurun_out/slab_tests_${TAG}.log 2>&1
echo "slab tests rc=$?"; tail -2 gpurun_out/slab_tests_${TAG}.log
for c in ${CONFIGS:-st1 st2 st3 st4 st5}; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_${c}_${TAG}.json 2> gpurun_out/bench_${c}_${TAG}.err
  echo "bench $c rc=$?"; cat gpurun_out/bench_${c}_${TAG}.json | head -c 1500; echo
done
if [ -z "$SKIP_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches_st3_${TAG}.csv python bench.py --config st3 --n 100000 --steps 2 --warmup 1 --profile \
    > gpurun_out/launches_st3_${TAG}.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pdg_slab_kernel -s 1 -c 1 \
    -o gpurun_out/prof_st3_${TAG} python bench.py --config st3 --n 100000 --steps 1 --warmup 1 --profile \
    > gpurun_out/ncu_st3_${TAG}.log 2>&1
echo "ncu full rc=$?"
fi
