#!/bin/bash
# Evidence capture for profiles/: bench lines (1M with CPU baseline, 10M u/c),
# ncu launch lists, ncu --set full captures of the top kernels at 1M and 10M.
set -x
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > gpurun_out/gpu.txt
( python -c "import bench; bench.load_mesh('u10m', 0)" > gpurun_out/gen_u10m.log 2>&1 ) &
( python -c "import bench; bench.load_mesh('c10m', 0)" > gpurun_out/gen_c10m.log 2>&1 ) &
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_u1m.json 2> gpurun_out/bench_u1m.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_u1m.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_u1m.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_u1m.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
   -k "regex:k_tri_pass|k_pair_pass|k_ruler_walk|k_repair_tips_seg|k_stitch_plain" -s 15 -c 5 \
   -o gpurun_out/prof_u1m python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_u1m.log 2>&1
wait
timeout 500 python bench.py --workload u10m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_u10m.json 2> gpurun_out/bench_u10m.err
timeout 500 python bench.py --workload c10m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c10m.json 2> gpurun_out/bench_c10m.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_u10m.csv \
   python bench.py --workload u10m --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_u10m.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
   -k "regex:k_tri_pass|k_pair_pass|k_ruler_walk|k_repair_tips_seg|k_stitch_plain" -s 15 -c 5 \
   -o gpurun_out/prof_u10m python bench.py --workload u10m --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_u10m.log 2>&1
timeout 900 python tools/partition_scaling.py --workload u10m --steps 5 > gpurun_out/scaling_u10m.json 2>&1
timeout 600 python tools/partition_scaling.py --workload u1m --steps 10 > gpurun_out/scaling_u1m.json 2>&1
ls -la gpurun_out
