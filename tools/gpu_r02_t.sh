#!/bin/bash
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
for v in default ab/prev.so; do
  if [ "$v" = default ]; then unset TERMESH_LIB_VARIANT; else export TERMESH_LIB_VARIANT=$PWD/$v; fi
  for w in ${WORKLOADS:-u10m c10m}; do
    timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python tools/bench_brief.py $v
  done
done
