#!/bin/bash
# 100M config (BASELINE.json configs[3]): tile-parallel exact Delaunay input,
# parity vs the oracle, bench line, seed-partition projection, launch list;
# then racecheck on the small cases.
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
{ nproc; free -g; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv; } > gpurun_out/host_100m.txt 2>&1
( time python -c "import bench; t = bench.load_mesh('u100m', 0); print(t.n_vertices, t.n_triangles)" ) > gpurun_out/gen_u100m.log 2>&1
timeout 900 python tools/check_100m.py --workload u1m --slices 0,7 --nslices 16 > gpurun_out/check_u1m.log 2>&1
timeout 2400 python tools/check_100m.py --workload u100m > gpurun_out/check_u100m.log 2>&1
timeout 1200 python bench.py --workload u100m --steps 10 --warmup 3 > gpurun_out/bench_u100m.json 2> gpurun_out/bench_u100m.err
timeout 1800 python tools/partition_scaling.py --workload u100m --steps 5 > gpurun_out/scaling_u100m.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_u100m.csv \
   python bench.py --workload u100m --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_u100m.log 2>&1
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 100000 python tools/sanitize_run.py > gpurun_out/sanitizer_racecheck.log 2>&1
ls -la gpurun_out
