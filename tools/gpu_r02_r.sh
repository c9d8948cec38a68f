#!/bin/bash
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
./build/dchk_fixed | tail -2
( python -c "import bench; bench.load_mesh('u100m', 0)" > gpurun_out/gen_u100m.log 2>&1 ) &
BISECT_WORKLOADS="c10m" bash tools/gpu_bisect.sh
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_r.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r.log
tail -3 gpurun_out/pytest_gpu_r.log
wait
BISECT_WORKLOADS="u100m" bash tools/gpu_bisect.sh
timeout 1200 python bench.py --workload u100m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_u100m_r.json 2> gpurun_out/bench_u100m_r.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_u10m_r.json 2> gpurun_out/bench_u10m_r.err
timeout 600 python bench.py --workload c10m --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c10m_r.json 2> gpurun_out/bench_c10m_r.err
cat gpurun_out/bench_u10m_r.json gpurun_out/bench_c10m_r.json gpurun_out/bench_u100m_r.json | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['config']['workload'], d['ms_per_step'], d['e2e']['ms_per_step'], d['parity']['match'])"
