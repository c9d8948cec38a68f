#!/bin/bash
# 10M configs (BASELINE.json configs 3 and 5): generation, bench, projected
# partition scaling, launch list + ncu full capture, full-size parity tests.
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
nproc > gpurun_out/big_host.txt; free -g >> gpurun_out/big_host.txt
( time python -c "import bench; bench.load_mesh('u10m', 0)" ) > gpurun_out/gen_u10m.log 2>&1 &
( time python -c "import bench; bench.load_mesh('c10m', 0)" ) > gpurun_out/gen_c10m.log 2>&1 &
wait
timeout 900 python bench.py --workload u10m --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_u10m.json 2> gpurun_out/bench_u10m.err
timeout 900 python bench.py --workload c10m --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c10m.json 2> gpurun_out/bench_c10m.err
timeout 600 python tools/partition_scaling.py --workload u10m --steps 5 > gpurun_out/scaling_u10m.json 2>&1
timeout 600 python tools/partition_scaling.py --workload u1m --steps 10 > gpurun_out/scaling_u1m.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_u10m.csv \
   python bench.py --workload u10m --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_u10m.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_tri_pass|k_pair_pass|k_ruler_walk" -s 3 -c 3 \
   -o gpurun_out/prof_u10m python bench.py --workload u10m --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full_u10m.log 2>&1
TERMESH_BIG=1 timeout 1500 python -m pytest tests/test_big.py -q -s > gpurun_out/pytest_big.log 2>&1
ls -la gpurun_out
