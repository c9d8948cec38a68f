#!/bin/bash
# Round-2 evidence session: GPU tests, smoke, bench lines (u10m default, c10m,
# u1m, reference arm), ncu launch list + --set full capture at 10M (raw metric
# dump for tools/ncu_summary.py), compute-sanitizer on small cases.
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > gpurun_out/gpu.txt
( python -c "import bench; bench.load_mesh('u10m', 0)" > gpurun_out/gen_u10m.log 2>&1 ) &
( python -c "import bench; bench.load_mesh('c10m', 0)" > gpurun_out/gen_c10m.log 2>&1 ) &
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
wait
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_u10m.json 2> gpurun_out/bench_u10m.err
timeout 600 python bench.py --workload c10m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c10m.json 2> gpurun_out/bench_c10m.err
timeout 600 python bench.py --workload u1m --steps 20 --warmup 5 > gpurun_out/bench_u1m.json 2> gpurun_out/bench_u1m.err
timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/bench_ref_u10m.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_u10m.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_u10m.log 2>&1
EXTRA=l1tex__m_l1tex2xbar_write_sectors_mem_global_op_atom.sum,l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,dram__bytes_read.sum,dram__bytes_write.sum
timeout 1500 ncu --set full --metrics $EXTRA --clock-control none --import-source on \
   -k "regex:k_tri_pass|k_pair_pass|k_ruler_walk|k_ruler_write|k_repair_tips|k_stitch_plain|k_chain" -s 26 -c 10 \
   -o gpurun_out/prof_u10m python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_u10m.log 2>&1
ncu -i gpurun_out/prof_u10m.ncu-rep --page raw --csv > gpurun_out/prof_u10m_raw.csv 2>&1
SAN_BIG=1 timeout 900 compute-sanitizer --tool memcheck --leak-check full python tools/sanitize_run.py > gpurun_out/sanitizer_memcheck.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_run.py > gpurun_out/sanitizer_racecheck.log 2>&1
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_run.py > gpurun_out/sanitizer_synccheck.log 2>&1
timeout 900 compute-sanitizer --tool initcheck python tools/sanitize_run.py > gpurun_out/sanitizer_initcheck.log 2>&1
ls -la gpurun_out
