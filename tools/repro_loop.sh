#!/bin/bash
# repeated bench runs, counting failures per env variant (run under gpurun)
mkdir -p gpurun_out; : > gpurun_out/repro.txt
IFS='|' read -ra VARS <<< "${AB_ENVS:--}"
for v in "${VARS[@]}"; do
  e="$v"; [ "$e" = "-" ] && e=""
  for w in ${WORKLOADS:-c10m}; do
    for i in $(seq ${REPS:-4}); do
      env $e timeout 300 python bench.py --workload $w --steps 30 --warmup 3 --no-cpu-baseline > /tmp/r.json 2> /tmp/r.err
      rc=$?
      echo "$v $w run$i rc=$rc $(grep -o 'Error: .*' /tmp/r.err | head -1)" >> gpurun_out/repro.txt
    done
  done
done
cat gpurun_out/repro.txt
