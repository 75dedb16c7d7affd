#!/bin/bash
# round-2 check: all GPU tests, smoke, 2-rank partitioned bench (gloo, shared GPU)
TAG=${1:-r02b}
mkdir -p gpurun_out
export PDG_JIT_CACHE=/tmp/pdg_jit
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/tests_${TAG}.log 2>&1
echo "tests rc=$?"; tail -25 gpurun_out/tests_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
echo "smoke rc=$?"; tail -2 gpurun_out/smoke_${TAG}.log
for c in cfg2 cfg4; do
PDG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --config $c --steps 3 --warmup 3 --no-e2e > gpurun_out/bench2_${c}_${TAG}.json 2> gpurun_out/bench2_${c}_${TAG}.err
echo "bench2 $c rc=$?"; cat gpurun_out/bench2_${c}_${TAG}.json | head -c 3000; tail -3 gpurun_out/bench2_${c}_${TAG}.err
done
