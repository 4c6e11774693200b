#!/bin/bash
# Build an A/B variant of the library: tools/build_variant.sh TAG -DFOO=1 ...
# -> paper_2502_08673_b200/libsatgrad_b200_TAG.so (A/B it with tools/ab.sh "<workloads>" base so:TAG)
set -e
tag=$1; shift
cd "$(dirname "$0")/../paper_2502_08673_b200/csrc"
nvcc -ccbin /usr/bin/g++ -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC,-O3 -Xptxas -O3 --expt-relaxed-constexpr "$@" -shared \
  -o ../libsatgrad_b200_$tag.so sgx_kernels.cu sgx_format.cu sgx_api.cpp sgx_layout.cpp sgx_layout_io.cpp sgx_drain.cpp sgx_extract.cpp \
  sgx_verify.cu sgx_jit.cpp sgx_exchange.cpp -ldl
