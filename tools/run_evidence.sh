#!/bin/bash
# Round evidence session (run at HEAD): tests, smoke, every bench line, the
# partitioned 2-rank path, the reference arm, ncu launch list + full captures,
# FP64 peaks with clocks, compute-sanitizer.   bash tools/run_evidence.sh r02x
TAG=${1:-r02x}
mkdir -p gpurun_out
export PDG_JIT_CACHE=/tmp/pdg_jit
nproc > gpurun_out/box_${TAG}.txt; lscpu | grep "Model name" >> gpurun_out/box_${TAG}.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv >> gpurun_out/box_${TAG}.txt
free -g >> gpurun_out/box_${TAG}.txt
if [ -z "$SKIP_TESTS" ]; then
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/tests_${TAG}.log 2>&1
echo "tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/tests_${TAG}.log | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
echo "smoke rc=$?"; tail -1 gpurun_out/smoke_${TAG}.log
fi
timeout 1200 python bench.py > gpurun_out/bench_cfg5_${TAG}.json 2> gpurun_out/bench_cfg5_${TAG}.err
echo "bench cfg5 rc=$?"; head -c 600 gpurun_out/bench_cfg5_${TAG}.json; echo
# the polydg-signature call at the headline scale (100 GB host CSR per call)
timeout 1200 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --e2e-api-max-gb 120 \
  > gpurun_out/bench_cfg5api_${TAG}.json 2> gpurun_out/bench_cfg5api_${TAG}.err
echo "bench cfg5 api rc=$? $(python -c "import json; d=json.load(open('gpurun_out/bench_cfg5api_${TAG}.json')); print(d.get('e2e_api'))" 2>&1 | tail -1)"
for c in cfg1 cfg2 cfg3p2 cfg3p3 cfg3 cfg3p5 cfg3p6 cfg4 st1 st2 st3 st4 st5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_${c}_${TAG}.json 2> gpurun_out/bench_${c}_${TAG}.err
  echo "bench $c rc=$? $(python -c "import json; d=json.load(open('gpurun_out/bench_${c}_${TAG}.json')); print(round(d['value']/1e6,2), 'M el/s', round(d['ms_per_step'],3), 'ms', round(d['roofline']['frac'],3), 'frac')" 2>&1 | tail -1)"
done
for c in cfg2 cfg3; do
  timeout 900 python bench.py --config $c --approach 1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/bench_${c}_a1_${TAG}.json 2> gpurun_out/bench_${c}_a1_${TAG}.err
  echo "bench $c A1 rc=$?"
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
echo "reference arm rc=$?"; head -c 300 gpurun_out/bench_ref_${TAG}.json; echo
for c in cfg2 cfg4; do
  PDG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29517 bench.py --gpus 2 --config $c --steps 5 --warmup 3 --no-e2e > gpurun_out/bench2_${c}_${TAG}.json 2> gpurun_out/bench2_${c}_${TAG}.err
  echo "2-rank $c rc=$? $(python -c "import json; d=json.load(open('gpurun_out/bench2_${c}_${TAG}.json')); print(d['scaling'], d['verified'], round(d['ms_per_step'],3))" 2>&1 | tail -1)"
done
# the N-rank path with 4 and 8 ranks time-sharing the one GPU (correctness of the split + gather)
for n in 4 8; do
  PDG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2952$n bench.py --gpus $n --config cfg2 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench${n}_cfg2_${TAG}.json 2> gpurun_out/bench${n}_cfg2_${TAG}.err
  echo "$n-rank cfg2 rc=$? $(python -c "import json; d=json.load(open('gpurun_out/bench${n}_cfg2_${TAG}.json')); print(d['scaling'], d['verified'], round(d['ms_per_step'],3), d['config']['max_local_elements'])" 2>&1 | tail -1)"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_cfg5_${TAG}.csv python bench.py --steps 2 --warmup 1 --profile \
    > gpurun_out/launches_cfg5_${TAG}.log 2>&1
echo "launches rc=$?"
for c in "cfg5 400000 pdg_jit_kernel" "cfg2 100000 pdg_jit_kernel" "cfg3p3 250000 pdg_jit_kernel" "cfg3 250000 pdg_jit_kernel" "cfg4 56 pdg_jit_kernel" "st3 100000 pdg_slab_kernel"; do
  set -- $c
  python bench.py --config $1 --n $2 --steps 1 --warmup 1 --profile > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 \
      -o gpurun_out/prof_${1}_${TAG} python bench.py --config $1 --n $2 --steps 1 --warmup 1 --profile \
      > gpurun_out/ncu_${1}_${TAG}.log 2>&1
  echo "ncu $1 rc=$?"
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/peaks_clocks_${TAG}.csv &
SMI=$!
./tools/fp64_peaks > gpurun_out/fp64_peaks_${TAG}.json 2>&1
kill $SMI
echo "peaks rc=$?"; cat gpurun_out/fp64_peaks_${TAG}.json | head -20
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python -m pytest tests/test_oracle_golden.py -m gpu -q \
     -k "engine and (cfg1_voronoi1000 or cube3_adr or cube4_advdiff3d or voronoi120_poisson_p4 or clusters6_poisson_p3)" \
     > gpurun_out/sanitizer_${tool}_${TAG}.log 2>&1
  echo "sanitizer $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitizer_${tool}_${TAG}.log | tail -1)"
done
