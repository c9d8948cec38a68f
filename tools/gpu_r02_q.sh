#!/bin/bash
# fixed dup-scan fast path + run staging (ab/staging.so): c10m/u100m runs, parity tests, A/B
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
( python -c "import bench; bench.load_mesh('u100m', 0)" > gpurun_out/gen_u100m.log 2>&1 ) &
BISECT_WORKLOADS="c10m" bash tools/gpu_bisect.sh
TERMESH_LIB_VARIANT=$PWD/ab/staging.so timeout 1500 python -m pytest tests/test_gpu_twin.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_q.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_q.log
tail -3 gpurun_out/pytest_q.log
STEPS=20 AB_WORKLOADS="u1m u10m" bash tools/ab_lib.sh
wait
cp gpurun_out/bisect.txt gpurun_out/bisect_c10m.txt
BISECT_WORKLOADS="u100m" bash tools/gpu_bisect.sh
