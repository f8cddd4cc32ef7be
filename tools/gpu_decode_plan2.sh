#!/bin/bash
# decode attention plan variants (tools/build_variant.sh builds)
mkdir -p gpurun_out
out=gpurun_out/dp_bench3.txt
: > $out
for v in old o20 o40 o60 o40pre; do
  echo "== $v" >> $out
  EMM_LIB_PATH=build/libemm_$v.so timeout 300 python tools/decode_bench.py >> $out 2>&1
done
