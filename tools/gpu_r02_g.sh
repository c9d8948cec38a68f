#!/bin/bash
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
timeout 1500 python -m pytest tests -q -m gpu -x -k "not test_10m" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
( time python -c "import bench; t = bench.load_mesh('u100m', 0)" ) > gpurun_out/gen_u100m.log 2>&1
timeout 600 python tools/spill_probe.py u100m > gpurun_out/spill_u100m.log 2>&1
timeout 1200 python bench.py --workload u100m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_u100m.json 2> gpurun_out/bench_u100m.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_u100m.csv \
   python bench.py --workload u100m --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_u100m.log 2>&1
timeout 1800 python tools/partition_scaling.py --workload u100m --steps 5 > gpurun_out/scaling_u100m.json 2>&1
timeout 2400 python tools/check_100m.py --workload u100m > gpurun_out/check_u100m.log 2>&1
ls -la gpurun_out
