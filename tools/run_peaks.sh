#!/bin/bash
# Measure FP64 peaks + host info on the GPU box. Output -> gpurun_out/peaks.*
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/peaks_clocks.csv &
SMI=$!
./tools/fp64_peak > gpurun_out/peaks_fp64.json 2>&1
python tools/dgemm_peak.py > gpurun_out/peaks_dgemm.json 2>&1
kill $SMI
nproc > gpurun_out/host_info.txt; lscpu | head -20 >> gpurun_out/host_info.txt; free -g >> gpurun_out/host_info.txt
nvidia-smi >> gpurun_out/host_info.txt
cat gpurun_out/peaks_fp64.json gpurun_out/peaks_dgemm.json
