#!/bin/bash
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_twin.py tests/test_distributed.py tests/test_gpu_post.py -x -q -m gpu 2>&1 | tail -2
for w in c10m; do timeout 600 python tools/bisect_c10m.py $w; done
WORKLOADS="u1m u10m c10m" bash tools/gpu_r02_t.sh
WORKLOADS="u10m c10m" bash tools/gpu_r02_t.sh
