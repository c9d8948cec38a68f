#!/bin/bash
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
python -c "import bench; bench.load_mesh('u10m', 0)" > gpurun_out/gen_u10m.log 2>&1
TRACE_WORKLOAD=u10m python tools/trace_long.py > gpurun_out/trace_u10m.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_u10m.csv \
   python bench.py --workload u10m --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_u10m.log 2>&1
