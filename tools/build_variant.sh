#!/bin/bash
# build/libemm_<name>.so: libemm with one source compiled with extra -D flags
# usage: tools/build_variant.sh prof -DATT_PROF=1            (attn_tc.cu)
#        SRC=decode_attn.cu tools/build_variant.sh t16 -DDA_TILE_KEYS=16
set -e
name=$1; shift
src=${SRC:-attn_tc.cu}
base=${src%.cu}
cd "$(dirname "$0")/.."
python -m paper_2507_10069_b200.build > /dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -I include -I paper_2507_10069_b200/csrc "$@" \
  -c paper_2507_10069_b200/csrc/$src -o build/emm/${base}_$name.o
objs=$(ls build/emm/*.cu.o build/emm/*.cpp.o | grep -v "/${base}.cu.o" | tr "\n" " ")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/libemm_$name.so $objs \
  build/emm/${base}_$name.o -lcudart_static
echo build/libemm_$name.so
