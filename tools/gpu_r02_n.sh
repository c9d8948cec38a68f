#!/bin/bash
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
timeout 900 python -m pytest tests/test_gpu_twin.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_n.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_n.log
tail -3 gpurun_out/pytest_n.log
STEPS=20 AB_WORKLOADS="u1m u10m" bash tools/ab_lib.sh
