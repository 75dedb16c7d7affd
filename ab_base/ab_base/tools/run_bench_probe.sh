set -x
nproc > gpurun_out/box.txt; free -g >> gpurun_out/box.txt; lscpu | grep "Model name" >> gpurun_out/box.txt
python bench.py --config cfg2 --steps 5 --warmup 3 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --config cfg2 --steps 2 --warmup 1 --profile > /dev/null 2>&1
ls -la /tmp/pdg_meshcache >> gpurun_out/box.txt
