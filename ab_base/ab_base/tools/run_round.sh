#!/bin/bash
# One GPU session: parity tests, smoke, the default bench line, the ncu launch
# list of the bench command and one full ncu capture of the element kernel.
#   tools/gpu.sh --timeout 3000 -- 'bash tools/run_round.sh r01b'
TAG=${1:-r01}
NPROF=${NPROF:-400000}
mkdir -p gpurun_out
export PDG_JIT_CACHE=/tmp/pdg_jit
nproc > gpurun_out/box_${TAG}.txt; lscpu | grep "Model name" >> gpurun_out/box_${TAG}.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv >> gpurun_out/box_${TAG}.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests_${TAG}.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/tests_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
echo "smoke rc=$?"; tail -2 gpurun_out/smoke_${TAG}.log
if [ -z "$SKIP_BENCH" ]; then
timeout 900 python bench.py > gpurun_out/bench_cfg5_${TAG}.json 2> gpurun_out/bench_cfg5_${TAG}.err
echo "bench rc=$?"; cat gpurun_out/bench_cfg5_${TAG}.json
fi
if [ -z "$SKIP_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_cfg5_${TAG}.csv python bench.py --steps 2 --warmup 1 --profile \
    > gpurun_out/launches_cfg5_${TAG}.log 2>&1
echo "launches rc=$?"
python bench.py --n $NPROF --steps 1 --warmup 1 --profile > /dev/null 2>&1   # warm the JIT + mesh caches
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pdg_jit_kernel -s 1 -c 1 \
    -o gpurun_out/prof_cfg5_${TAG} python bench.py --n $NPROF --steps 1 --warmup 1 --profile \
    > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu full rc=$?"
fi
