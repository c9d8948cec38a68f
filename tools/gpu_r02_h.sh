#!/bin/bash
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
timeout 1500 python -m pytest tests/test_distributed.py -q -m gpu -x > gpurun_out/pytest_dist.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_dist.log
timeout 900 python tools/partition_scaling.py --workload u10m --steps 6 --split > gpurun_out/scaling_split_u10m.json 2>&1
( time python -c "import bench; t = bench.load_mesh('u100m', 0)" ) > gpurun_out/gen_u100m.log 2>&1
timeout 2400 python tools/partition_scaling.py --workload u100m --steps 3 --split > gpurun_out/scaling_split_u100m.json 2>&1
ls -la gpurun_out
