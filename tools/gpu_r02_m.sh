#!/bin/bash
# single-pass labels on the host entry: parity tests, then A/B of the e2e against two-pass
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
timeout 900 python -m pytest tests/test_gpu_twin.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_m.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_m.log
tail -3 gpurun_out/pytest_m.log
STEPS=20 AB_WORKLOADS="u1m u10m" AB_ENVS="-|TERMESH_LABEL_ONE=0" bash tools/ab_env.sh
