#!/bin/bash
# tests + 1M bench, then the 10M configs (bench + full-size parity)
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
( python -c "import bench; bench.load_mesh('u10m', 0)" > gpurun_out/gen_u10m.log 2>&1 ) &
( python -c "import bench; bench.load_mesh('c10m', 0)" > gpurun_out/gen_c10m.log 2>&1 ) &
timeout 900 python -m pytest tests -q -m gpu -x --timeout=300 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 240 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
wait
timeout 420 python bench.py --workload u10m --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_u10m.json 2> gpurun_out/bench_u10m.err
timeout 420 python bench.py --workload c10m --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c10m.json 2> gpurun_out/bench_c10m.err
if [ -n "$BIGTEST" ]; then TERMESH_BIG=1 timeout 1500 python -m pytest tests/test_big.py -q -s > gpurun_out/pytest_big.log 2>&1; fi
if [ -n "$TRACE" ]; then python tools/trace_long.py > gpurun_out/trace.txt 2>&1; fi
tail -2 gpurun_out/pytest_gpu.log
