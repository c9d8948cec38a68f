#!/bin/bash
# full ncu capture of selected kernels (run under gpurun): NCU_KERNELS regex, NCU_SKIP, NCU_COUNT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${NCU_KERNELS:-k_tri_pass}" -s ${NCU_SKIP:-6} -c ${NCU_COUNT:-2} \
   -o gpurun_out/${NCU_OUT:-prof} python bench.py --steps 1 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
