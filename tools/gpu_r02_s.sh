#!/bin/bash
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_twin.py -x -q -m gpu 2>&1 | tail -2
unset TERMESH_LIB_VARIANT; timeout 600 python tools/bisect_c10m.py c10m
STEPS=20 AB_WORKLOADS="u1m u10m c10m" bash tools/ab_lib.sh
