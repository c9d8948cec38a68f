#!/bin/bash
# parity tests + 1M / 10M bench lines (run under gpurun)
mkdir -p gpurun_out
timeout ${TEST_TIMEOUT:-900} python -m pytest tests -q -m gpu -x --timeout=300 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for w in u1m u10m c10m; do
  timeout 300 python bench.py --workload $w --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_$w.json').readline()); print('$w', d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['frac'])"
done
