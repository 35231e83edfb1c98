#!/bin/bash
# ncu evidence for the bench workload: launch list of one sweep + full capture of one fused step.
# usage: tools/prof_run.sh TAG   (outputs gpurun_out/launches_TAG.csv, gpurun_out/prof_TAG.ncu-rep)
TAG=${1:-r01}
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"chase|step_kernel|bulk_update" -c 440 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_list_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"step_kernel" -s 200 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
tail -2 gpurun_out/plain_$TAG.log | cut -c1-300
