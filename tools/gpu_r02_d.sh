#!/bin/bash
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
timeout 900 python tools/delaunay_diff.py 1000000 0 > gpurun_out/delaunay_diff_1m.log 2>&1
( time python -c "import bench; t = bench.load_mesh('u100m', 0)" ) > gpurun_out/gen_u100m.log 2>&1
timeout 900 python tools/long_items.py u100m > gpurun_out/long_items_u100m.log 2>&1
timeout 600 python tools/long_items.py u10m > gpurun_out/long_items_u10m.log 2>&1
AB_ENVS="-|TERMESH_NO_XY32=1" AB_WORKLOADS="u10m u1m" STEPS=20 bash tools/ab_env.sh > gpurun_out/ab_xy32.log 2>&1
ls -la gpurun_out
