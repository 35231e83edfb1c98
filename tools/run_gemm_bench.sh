#!/bin/bash
# isolated update-kernel timings (tools/gemm_bench.cu variants): interior windows, even and odd w0
for b in tools/gemm_bench_base tools/gemm_bench_nostore; do
  echo "== $b"
  $b 20000 18 96 15 8000 20 2>/dev/null
  $b 20000 18 96 15 8001 20 2>/dev/null
done
