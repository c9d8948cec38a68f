#!/bin/bash
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
for e in 16 64 148; do
  for w in u1m u10m c10m; do
    TERMESH_PINCH2_BLOCKS=$e timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python tools/bench_brief.py p2=$e | cut -c1-60
  done
done
TERMESH_PINCH2_BLOCKS=148 TERMESH_STAMPS=1 timeout 300 python tools/trace_step.py u10m | tail -6
