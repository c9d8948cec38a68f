#!/bin/bash
# A/B timing of library variants (run under gpurun): default build vs each ab/*.so,
# with the bench line's parity verdict and the label-pass kernel times.
mkdir -p gpurun_out; : > gpurun_out/ab.txt
export TERMESH_CACHE=${TERMESH_CACHE:-/tmp/termesh_cache}
for w in ${AB_WORKLOADS:-u1m u10m}; do python -c "import bench; bench.load_mesh('$w', 0)" > /dev/null 2>&1; done
for rep in $(seq ${AB_REPS:-2}); do
for v in default ab/*.so; do
  for w in ${AB_WORKLOADS:-u1m u10m}; do
    if [ "$v" = default ]; then unset TERMESH_LIB_VARIANT; else export TERMESH_LIB_VARIANT=$PWD/$v; fi
    timeout 300 python bench.py --workload $w --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.readline()); k=d['kernels']; print('$v', '$w', d['ms_per_step'], d['e2e']['ms_per_step'], 'parity', d['parity']['match'], ' '.join(f'{n}={v[\"ms\"]:.3f}' for n,v in k.items() if n.startswith(tuple(__import__('os').environ.get('AB_KERNELS','label trav_r').split()))))" >> gpurun_out/ab.txt
  done
done; done
cat gpurun_out/ab.txt
