#!/bin/bash
# K-loop variant microbenchmark (tools/gemm_bench.cu built with -DHQR_KLOOP=v): interior windows
for b in tools/gemm_bench_k_base tools/gemm_bench_k0 tools/gemm_bench_k1 tools/gemm_bench_k2 tools/gemm_bench_k3; do
  echo "== $b"
  $b 20000 18 96 15 8000 20 2>/dev/null
done
