#!/bin/bash
# balanced seed ranges: parity tests + projected split-label scaling with measured-cost rebalancing (u10m, u100m)
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
timeout 900 python -m pytest tests -q -m gpu -x -k "distributed or split" > gpurun_out/pytest_dist.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_dist.log
tail -2 gpurun_out/pytest_dist.log
timeout 900 python tools/partition_scaling.py --workload u10m --steps 6 --split --balance 3 --segments > gpurun_out/scaling_bal_u10m.json 2> gpurun_out/scaling_bal_u10m.err
( time python -c "import bench; t = bench.load_mesh('u100m', 0)" ) > gpurun_out/gen_u100m.log 2>&1
timeout 2400 python tools/partition_scaling.py --workload u100m --steps 3 --split --balance 3 --segments > gpurun_out/scaling_bal_u100m.json 2> gpurun_out/scaling_bal_u100m.err
ls -la gpurun_out
