#!/bin/bash
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
for v in default ab/noxy.so ab/notable.so ab/noboth.so; do
  if [ "$v" = default ]; then unset TERMESH_LIB_VARIANT; else export TERMESH_LIB_VARIANT=$PWD/$v; fi
  timeout 600 python tools/label_ab.py u10m >> gpurun_out/label_ab.log 2>&1
done
unset TERMESH_LIB_VARIANT
timeout 900 python tools/k0_sort_ab.py u10m > gpurun_out/k0_sort_ab.log 2>&1
timeout 900 python tools/partition_scaling.py --workload u10m --steps 6 --split > gpurun_out/scaling_split_u10m.json 2>&1
ls -la gpurun_out
