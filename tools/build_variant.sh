#!/bin/bash
# Build a compile-time variant of the library: tools/build_variant.sh NAME -DFOO=1 ...
# -> paper_0904_3151_b200/_native/libeg_NAME.so (select with EG_LIB_PATH)
set -e
name=$1; shift
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared "$@" \
  -o paper_0904_3151_b200/_native/libeg_$name.so paper_0904_3151_b200/csrc/capi.cu
echo built libeg_$name.so
