#!/bin/bash
# full evaluation on the GPU box: gpu tests, bench (all keys), reference arm, ncu launch list
# usage: tools/round_eval.sh TAG
TAG=${1:-r01}
timeout -s KILL 700 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; tail -2 gpurun_out/pytest_gpu_$TAG.log
timeout -s KILL 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1; tail -1 gpurun_out/bench_$TAG.log | cut -c1-200
timeout -s KILL 300 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.log 2>&1; tail -1 gpurun_out/bench_ref_$TAG.log | cut -c1-200
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"chase|step_kernel|bulk_update" -c 20 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_list_$TAG.log 2>&1
echo "launch list rows: $(wc -l < gpurun_out/launches_$TAG.csv)"
