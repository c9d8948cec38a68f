#!/bin/bash
# A/B timing of library variants (run under gpurun): default build vs each ab/*.so
mkdir -p gpurun_out; : > gpurun_out/ab.txt
for rep in 1 2; do
for v in default ab/*.so; do
  for w in ${AB_WORKLOADS:-u1m u10m}; do
    if [ "$v" = default ]; then unset TERMESH_LIB_VARIANT; else export TERMESH_LIB_VARIANT=$PWD/$v; fi
    timeout 300 python bench.py --workload $w --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.readline()); k=d['kernels']; print('$v', '$w', d['ms_per_step'], d['e2e']['ms_per_step'], ' '.join(f'{n}={v[\"ms\"]:.3f}' for n,v in k.items()))" >> gpurun_out/ab.txt
  done
done; done
cat gpurun_out/ab.txt
