#!/bin/bash
# Checked build of the library (bounds asserts in the epoch kernel, epoch.cu
# BCT_CHECK): paper_1709_00953_b200/_lib/libblockct_cuda_checked.so.  Run the
# GPU tests against it with
#   BCT_LIB=paper_1709_00953_b200/_lib/libblockct_cuda_checked.so python -m pytest tests -m gpu
set -e
cd "$(dirname "$0")/.."
tools/build_variant.sh checked -DBCT_CHECK=1
