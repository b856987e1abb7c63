#!/bin/bash
# Diagnostic build of the library with the selection/append/pass %globaltimer
# marks (-DGTC_SEL_TRACE): paper_2111_14991_b200/libgridtune_b200_trace.so
set -e
cd "$(dirname "$0")/../paper_2111_14991_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++20 -Xcompiler -fPIC -Xcompiler -O3 -shared \
  -DGTC_SEL_TRACE -I ../../include -o ../libgridtune_b200_trace.so \
  gtc_kernels.cu enum_kernels.cu gtc_capi.cu bo_host.cpp restriction.cpp cache_host.cpp comm.cpp -lcudart -ldl
