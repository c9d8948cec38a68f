#!/bin/bash
# Round evidence for profiles/<tag>: bench lines (u10m default + CPU baseline,
# c10m, u1m, u100m), reference arm, launch lists, ncu --set full at 10M,
# seed-partition projections, 100M parity, GPU Delaunay check, sanitizers.
set -x
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > gpurun_out/gpu.txt
( python -c "import bench; bench.load_mesh('c10m', 0)" > gpurun_out/gen_c10m.log 2>&1 ) &
( python -c "import bench; bench.load_mesh('u1m', 0)" > gpurun_out/gen_u1m.log 2>&1 ) &
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
wait
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_u10m.json 2> gpurun_out/bench_u10m.err
timeout 600 python bench.py --workload c10m --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c10m.json 2> gpurun_out/bench_c10m.err
timeout 600 python bench.py --workload u1m --steps 20 --warmup 5 > gpurun_out/bench_u1m.json 2> gpurun_out/bench_u1m.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_u10m.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_u10m.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_u10m.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_u1m.csv \
   python bench.py --workload u1m --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_u1m.log 2>&1
EXTRA=l1tex__m_l1tex2xbar_write_sectors_mem_global_op_atom.sum,l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,dram__bytes_read.sum,dram__bytes_write.sum
timeout 1500 ncu --set full --metrics $EXTRA --clock-control none --import-source on \
   -k "regex:k_tri_pass|k_pair_pass|k_ruler_walk|k_ruler_write|k_repair_tips|k_stitch|k_chain|k_classify" -s 26 -c 12 \
   -o gpurun_out/prof_u10m python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_u10m.log 2>&1
ncu -i gpurun_out/prof_u10m.ncu-rep --page raw --csv > gpurun_out/prof_u10m_raw.csv 2>&1
timeout 900 python tools/partition_scaling.py --workload u10m --steps 10 > gpurun_out/scaling_u10m.json 2>&1
timeout 900 python tools/partition_scaling.py --workload u10m --steps 6 --split --balance 3 --segments > gpurun_out/scaling_split_u10m.json 2>&1
TRACE_WORKLOAD=u1m timeout 600 python tools/trace_long.py > gpurun_out/trace_u1m.log 2>&1
TERMESH_STAMPS=1 timeout 600 python tools/trace_step.py u10m > gpurun_out/trace_step.log 2>&1
( time python -c "import bench; t = bench.load_mesh('u100m', 0)" ) > gpurun_out/gen_u100m.log 2>&1
timeout 1200 python bench.py --workload u100m --steps 10 --warmup 3 > gpurun_out/bench_u100m.json 2> gpurun_out/bench_u100m.err
timeout 1800 python tools/partition_scaling.py --workload u100m --steps 5 > gpurun_out/scaling_u100m.json 2>&1
timeout 2400 python tools/partition_scaling.py --workload u100m --steps 3 --split --balance 3 --segments > gpurun_out/scaling_split_u100m.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_u100m.csv \
   python bench.py --workload u100m --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_u100m.log 2>&1
timeout 2400 python tools/check_100m.py --workload u100m > gpurun_out/check_u100m.log 2>&1
ls -la gpurun_out
