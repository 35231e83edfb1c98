#!/bin/bash
# Round-2 profiling on the GPU box: the ncu launch list of the bench command (the persistent fused
# kernel's per-launch time, DRAM bytes and DMMA pipe activity) and one `--set full` capture of a
# mid-sweep step of the same kernel code launched per step (HQR_PER_STEP=1 needs the tuning build,
# tools/build_variant.sh paper_2007_03576_b200/libhqr_timing.so "-DHQR_TIMING -DHQR_TUNING" is not
# used here: libhqr_tuning.so = "-DHQR_TUNING" only, no timers).
# usage: tools/prof_r02.sh TAG
TAG=${1:-r02}
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second \
  --clock-control none -k regex:"chase|step_kernel" -c 8 --csv --log-file gpurun_out/ncu_launches_$TAG.csv $CMD > gpurun_out/ncu_list_$TAG.log 2>&1
echo "launch list rc=$? rows=$(wc -l < gpurun_out/ncu_launches_$TAG.csv)"
HQR_LIB=$PWD/paper_2007_03576_b200/libhqr_tuning.so HQR_PER_STEP=1 ncu --set full --clock-control none --import-source on \
  -k regex:"step_kernel" -s 200 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full capture rc=$?"
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/srccs_$TAG.csv 2>/dev/null
ls -la gpurun_out/ | grep $TAG
