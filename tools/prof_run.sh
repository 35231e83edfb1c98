#!/bin/bash
# ncu evidence for the bench workload: launch list of one sweep + full capture of one step's kernels.
# usage: tools/prof_run.sh TAG   (outputs gpurun_out/launches_TAG.csv, gpurun_out/prof_TAG.ncu-rep)
TAG=${1:-r01}
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"chase|left_|right_" -c 1800 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_list_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"chase|left_|right_" -s 120 -c 4 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
tail -2 gpurun_out/plain_$TAG.log
