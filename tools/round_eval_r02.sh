#!/bin/bash
# Round-2 evaluation on the GPU box: the default bench line (configs[3], all keys), the other
# workloads, the reference arm and the ncu launch list of the default bench command.
T=${1:-r02}
python bench.py > gpurun_out/bench_${T}_cfg3.log 2>&1; tail -1 gpurun_out/bench_${T}_cfg3.log | cut -c1-200
python bench.py --config 2 --steps 10 --warmup 3 > gpurun_out/bench_${T}_cfg2.log 2>&1; tail -1 gpurun_out/bench_${T}_cfg2.log | cut -c1-200
python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${T}_cfg4.log 2>&1; tail -1 gpurun_out/bench_${T}_cfg4.log | cut -c1-200
python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${T}_cfg1.log 2>&1; tail -1 gpurun_out/bench_${T}_cfg1.log | cut -c1-200
python bench.py --sweeps 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${T}_sweeps4.log 2>&1; tail -1 gpurun_out/bench_${T}_sweeps4.log | cut -c1-200
python bench.py --workload hess --n 10000 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${T}_hess.log 2>&1; tail -1 gpurun_out/bench_${T}_hess.log | cut -c1-200
python bench.py --impl reference > gpurun_out/bench_${T}_ref.log 2>&1; tail -1 gpurun_out/bench_${T}_ref.log | cut -c1-200
