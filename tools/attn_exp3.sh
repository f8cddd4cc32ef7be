#!/bin/bash
# suspend-hint waits (no spinning) in the attention kernels: base vs variants
for v in base ws wsa wsap7 base; do
  if [ $v = base ]; then L=""; else L="EMM_LIB_PATH=build/libemm_$v.so"; fi
  echo "== $v"
  env $L timeout 300 python tools/attn_bench.py 2>&1 | grep -v "^c2\|^vit-clip"
done
