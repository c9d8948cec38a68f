#!/bin/bash
# A/B timing of env settings (run under gpurun): AB_ENVS="A=1 B=2|C=3" ('|' separates variants; '-' = none)
mkdir -p gpurun_out; : > gpurun_out/ab.txt
IFS='|' read -ra VARS <<< "${AB_ENVS:--}"
for rep in 1 2; do
for v in "${VARS[@]}"; do
  for w in ${AB_WORKLOADS:-u1m u10m}; do
    e="$v"; [ "$e" = "-" ] && e=""
    env $e timeout 300 python bench.py --workload $w --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.readline()); k=d['kernels']; print('$v', '$w', d['ms_per_step'], d['e2e']['ms_per_step'], ' '.join(f'{n}={v[\"ms\"]:.3f}' for n,v in k.items()))" >> gpurun_out/ab.txt
  done
done; done
cat gpurun_out/ab.txt
