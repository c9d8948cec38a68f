#!/bin/bash
# GPU tests + sanitizers + launch-count probe (no big inputs).
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 300 python tools/launch_probe.py > gpurun_out/launch_probe.log 2>&1
SAN_BIG=1 timeout 900 compute-sanitizer --tool memcheck --leak-check full python tools/sanitize_run.py > gpurun_out/sanitizer_memcheck.log 2>&1
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 100000 python tools/sanitize_run.py > gpurun_out/sanitizer_racecheck.log 2>&1
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_run.py > gpurun_out/sanitizer_synccheck.log 2>&1
timeout 900 compute-sanitizer --tool initcheck python tools/sanitize_run.py > gpurun_out/sanitizer_initcheck.log 2>&1
ls -la gpurun_out
