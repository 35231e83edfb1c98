#!/bin/bash
# bench + one ncu --set full capture (with source) of a mid-sweep fused step kernel.
# usage: tools/prof_step.sh TAG
TAG=${1:-x}
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_prof_$TAG.log 2>&1
tail -1 gpurun_out/bench_prof_$TAG.log | cut -c1-400
# the full capture takes one step's launch of the same kernel (HQR_PER_STEP=1: a launch per step; the
# bench's persistent launch spans the whole sweep)
HQR_PER_STEP=1 ncu --set full --clock-control none --import-source on -k regex:"step_kernel" -s 200 -c 1 -o gpurun_out/prof_$TAG \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_$TAG.log 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/srccs_$TAG.csv 2>/dev/null
