#!/bin/bash
# mid-round check: all GPU tests, u10m + u100m bench lines, ncu of the repair and label kernels at 10M
mkdir -p gpurun_out
export TERMESH_CACHE=/tmp/termesh_cache
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_o.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_o.log
tail -3 gpurun_out/pytest_gpu_o.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_u10m_o.json 2> gpurun_out/bench_u10m_o.err
EXTRA=l1tex__m_l1tex2xbar_write_sectors_mem_global_op_atom.sum,l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 1200 ncu --set full --metrics $EXTRA --clock-control none --import-source on \
   -k "regex:k_tri_pass|k_pair_pass|k_repair_tips$|k_ruler_write$|k_ruler_walk$" -s 10 -c 6 \
   -o gpurun_out/prof_u10m_o python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_u10m_o.log 2>&1
ncu -i gpurun_out/prof_u10m_o.ncu-rep --page raw --csv > gpurun_out/prof_u10m_o_raw.csv 2>&1
( time python -c "import bench; t = bench.load_mesh('u100m', 0)" ) > gpurun_out/gen_u100m.log 2>&1
timeout 1200 python bench.py --workload u100m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_u100m_o.json 2> gpurun_out/bench_u100m_o.err
cat gpurun_out/bench_u10m_o.json gpurun_out/bench_u100m_o.json | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['config']['workload'], d['ms_per_step'], d['e2e']['ms_per_step'], d['parity'])"
