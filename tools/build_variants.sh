#!/bin/bash
# Build tuning variants of the library into build/var_<name>.so (select one at
# run time with FMHA_B200_LIB=build/var_<name>.so).  Usage: tools/build_variants.sh name "-DFOO=1 ..." ...
set -e
cd "$(dirname "$0")/.."
P=paper_2312_11918_b200
SRCS="$P/csrc/fmha_api.cu $P/csrc/fmha_reference.cu $P/csrc/fmha_host.cpp $P/csrc/fmha_io.cpp"
mkdir -p build
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC \
    --expt-relaxed-constexpr $defs -shared -o build/var_$name.so $SRCS -lpthread &
done
wait
