#!/bin/bash
# Profiling: build a variant of the library with extra -D flags for epoch.cu,
#   tools/build_variant.sh NAME -DFOO=1 ...
# -> paper_1709_00953_b200/_lib/libblockct_cuda_NAME.so; select it with
# BCT_LIB=paper_1709_00953_b200/_lib/libblockct_cuda_NAME.so (same-box A/B).
set -e
cd "$(dirname "$0")/../paper_1709_00953_b200/csrc"
make -s >/dev/null
NAME=$1; shift
NVCC=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
$NVCC $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC "$@" -c epoch.cu -o /tmp/epoch_$NAME.o
$NVCC $ARCH -shared -o ../_lib/libblockct_cuda_$NAME.so /tmp/epoch_$NAME.o ../_lib/builder.o \
    ../_lib/layout.o ../_lib/sampler.o ../_lib/baseline.o ../_lib/api.o
echo ../_lib/libblockct_cuda_$NAME.so
