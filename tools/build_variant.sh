#!/bin/bash
# build/libemm_<name>.so: libemm with attn_tc.cu compiled with extra -D flags
# usage: tools/build_variant.sh prof -DATT_PROF=1
set -e
name=$1; shift
cd "$(dirname "$0")/.."
python -m paper_2507_10069_b200.build > /dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -I include -I paper_2507_10069_b200/csrc "$@" \
  -c paper_2507_10069_b200/csrc/attn_tc.cu -o build/emm/attn_tc_$name.o
objs=$(ls build/emm/*.o | grep -v "attn_tc" | tr '\n' ' ')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/libemm_$name.so $objs \
  build/emm/attn_tc_$name.o -lcudart_static
echo build/libemm_$name.so
