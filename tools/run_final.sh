#!/bin/bash
# Round-end evidence session: all GPU tests, smoke, the default bench line,
# every config line (cfg1-4, slabs st1-5, Approach 1 on cfg2/cfg3), the ncu
# launch list of the bench command and ncu --set full captures of the
# element kernel (cfg5-shaped 400k cells) and the slab kernel (st3, 100k).
TAG=${1:-final}
mkdir -p gpurun_out
export PDG_JIT_CACHE=/tmp/pdg_jit
nproc > gpurun_out/box_${TAG}.txt; lscpu | grep "Model name" >> gpurun_out/box_${TAG}.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv >> gpurun_out/box_${TAG}.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/tests_${TAG}.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/tests_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
echo "smoke rc=$?"; tail -1 gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_cfg5_${TAG}.json 2> gpurun_out/bench_cfg5_${TAG}.err
echo "bench cfg5 rc=$?"
for c in cfg1 cfg2 cfg3 cfg4 st1 st2 st3 st4 st5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_${c}_${TAG}.json 2> gpurun_out/bench_${c}_${TAG}.err
  echo "bench $c rc=$?"
done
for c in cfg2 cfg3; do
  timeout 900 python bench.py --config $c --approach 1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/bench_${c}_a1_${TAG}.json 2> gpurun_out/bench_${c}_a1_${TAG}.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
echo "reference arm rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_cfg5_${TAG}.csv python bench.py --steps 2 --warmup 1 --profile \
    > gpurun_out/launches_cfg5_${TAG}.log 2>&1
echo "launches rc=$?"
python bench.py --n 400000 --steps 1 --warmup 1 --profile > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pdg_jit_kernel -s 1 -c 1 \
    -o gpurun_out/prof_cfg5_${TAG} python bench.py --n 400000 --steps 1 --warmup 1 --profile \
    > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu cfg5 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pdg_slab_kernel -s 1 -c 1 \
    -o gpurun_out/prof_st3_${TAG} python bench.py --config st3 --n 100000 --steps 1 --warmup 1 --profile \
    > gpurun_out/ncu_st3_${TAG}.log 2>&1
echo "ncu st3 rc=$?"
