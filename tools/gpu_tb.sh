#!/bin/bash
# tests + bench only (run under gpurun)
mkdir -p gpurun_out
timeout ${TEST_TIMEOUT:-900} python -m pytest tests -q -m gpu -x --timeout=300 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 240 python bench.py --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/pytest_gpu.log
