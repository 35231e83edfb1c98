#!/bin/bash
# Build an alternative copy of libhqr_b200.so with extra nvcc flags (timing / tuning / debugging
# builds; never the product library).  usage: tools/build_variant.sh OUT.so "-DHQR_TIMING -DHQR_TUNING"
set -e
cd "$(dirname "$0")/.."
OUT=$1; shift
NCCL=$(python -c "import nvidia.nccl, os; print(list(nvidia.nccl.__path__)[0])")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -cudart shared --expt-relaxed-constexpr -I $NCCL/include $@ -o $OUT \
  paper_2007_03576_b200/csrc/{hqr_api,chase,update,step,qz,qriter}.cu -L $NCCL/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL/lib
