#!/bin/bash
# Round-2 first session: host probe, GPU tests, 10M generation timing, u10m bench.
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
{ nproc; free -g; df -h /tmp; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv; } > gpurun_out/host.txt 2>&1
( time python -c "import bench; bench.load_mesh('u10m', 0)" ) > gpurun_out/gen_u10m.log 2>&1 &
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
wait
timeout 600 python bench.py --workload u10m --steps 10 --warmup 3 > gpurun_out/bench_u10m.json 2> gpurun_out/bench_u10m.err
ls -la gpurun_out
