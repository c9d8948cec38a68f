#!/bin/bash
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
AB_WORKLOADS="u1m u10m" STEPS=20 bash tools/ab_lib.sh > gpurun_out/ab_lib.log 2>&1
( time python -c "import bench; t = bench.load_mesh('u100m', 0)" ) > gpurun_out/gen_u100m.log 2>&1
timeout 600 python tools/spill_probe.py u100m > gpurun_out/spill_u100m.log 2>&1
timeout 600 python tools/spill_probe.py u10m > gpurun_out/spill_u10m.log 2>&1
ls -la gpurun_out
