#!/bin/bash
# Round-2 (final: K loop, QZ far-right deferral, trimmed uploads, aligned tiles) evaluation on the GPU box: full GPU tests, the default bench line (configs[3], all
# keys), the other workloads, the reference arm, and the ncu launch list of the default command.
T=${1:-r02d}
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_${T}.log 2>&1; tail -1 gpurun_out/pytest_gpu_${T}.log
python bench.py > gpurun_out/bench_${T}_cfg3.log 2>&1; tail -1 gpurun_out/bench_${T}_cfg3.log | cut -c1-160
python bench.py --config 2 --steps 10 --warmup 3 > gpurun_out/bench_${T}_cfg2.log 2>&1; tail -1 gpurun_out/bench_${T}_cfg2.log | cut -c1-160
python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${T}_cfg4.log 2>&1; tail -1 gpurun_out/bench_${T}_cfg4.log | cut -c1-160
python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${T}_cfg1.log 2>&1; tail -1 gpurun_out/bench_${T}_cfg1.log | cut -c1-160
python bench.py --sweeps 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${T}_sweeps4.log 2>&1; tail -1 gpurun_out/bench_${T}_sweeps4.log | cut -c1-160
python bench.py --workload hess --n 10000 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${T}_hess.log 2>&1; tail -1 gpurun_out/bench_${T}_hess.log | cut -c1-160
python bench.py --workload qz --steps 5 --warmup 3 > gpurun_out/bench_${T}_qz.log 2>&1; tail -1 gpurun_out/bench_${T}_qz.log | cut -c1-160
python bench.py --workload qriter --steps 3 --warmup 1 > gpurun_out/bench_${T}_qriter.log 2>&1; tail -1 gpurun_out/bench_${T}_qriter.log | cut -c1-160
python bench.py --impl reference > gpurun_out/bench_${T}_ref.log 2>&1; tail -1 gpurun_out/bench_${T}_ref.log | cut -c1-160
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none -k regex:"chase|step_kernel" -c 8 --csv --log-file gpurun_out/ncu_launches_${T}.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_list_${T}.log 2>&1
echo "ncu rc=$? rows=$(wc -l < gpurun_out/ncu_launches_${T}.csv)"
bash tools/prof_r02.sh ${T}p
