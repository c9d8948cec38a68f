#!/bin/bash
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
AB_ENVS="-|TERMESH_NO_NARROW=1" AB_WORKLOADS="u1m u10m" STEPS=20 bash tools/ab_env.sh > gpurun_out/ab_narrow.log 2>&1
ls -la gpurun_out
