#!/bin/bash
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
TRACE_WORKLOAD=u1m timeout 600 python tools/trace_long.py > gpurun_out/trace_u1m.log 2>&1
TRACE_WORKLOAD=u10m timeout 900 python tools/trace_long.py > gpurun_out/trace_u10m.log 2>&1
ls -la gpurun_out
