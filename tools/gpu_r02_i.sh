#!/bin/bash
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
( time python -c "import bench; t = bench.load_mesh('u100m', 0)" ) > gpurun_out/gen_u100m.log 2>&1
timeout 1200 python bench.py --workload u100m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_u100m.json 2> gpurun_out/bench_u100m.err
timeout 600 python tools/spill_probe.py u100m > gpurun_out/spill_u100m.log 2>&1
timeout 2400 python tools/partition_scaling.py --workload u100m --steps 3 --split > gpurun_out/scaling_split_u100m.json 2>&1
timeout 900 python tools/partition_scaling.py --workload u10m --steps 6 --split > gpurun_out/scaling_split_u10m.json 2>&1
AB_ENVS="-" AB_WORKLOADS="u1m u10m" STEPS=20 bash tools/ab_env.sh > gpurun_out/ab_base.log 2>&1
ls -la gpurun_out
