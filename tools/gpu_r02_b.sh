#!/bin/bash
# GPU tests + 100M bench/scaling after the huge-item fixes, 10M bench + ncu.
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
( python -c "import bench; bench.load_mesh('u10m', 0)" > gpurun_out/gen_u10m.log 2>&1 ) &
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
wait
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_u10m.json 2> gpurun_out/bench_u10m.err
( time python -c "import bench; t = bench.load_mesh('u100m', 0)" ) > gpurun_out/gen_u100m.log 2>&1
timeout 1200 python bench.py --workload u100m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_u100m.json 2> gpurun_out/bench_u100m.err
timeout 1800 python tools/partition_scaling.py --workload u100m --steps 5 > gpurun_out/scaling_u100m.json 2>&1
timeout 900 python tools/partition_scaling.py --workload u10m --steps 10 > gpurun_out/scaling_u10m.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_u100m.csv \
   python bench.py --workload u100m --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_u100m.log 2>&1
timeout 2400 python tools/check_100m.py --workload u100m > gpurun_out/check_u100m.log 2>&1
ls -la gpurun_out
