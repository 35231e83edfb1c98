#!/bin/bash
# isolated update-kernel timings (tools/gemm_bench.cu variants)
for b in tools/gemm_bench_*; do
  echo "== $b"
  $b 20000 18 96 15 8000 20
  $b 20000 18 96 15 1000 20
done
