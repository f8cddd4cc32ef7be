#!/bin/bash
# single-tile kernel (windowed ViT layers): Q double-buffered (next item's Q in flight)
for v in base q2 base q2; do
  if [ $v = base ]; then L=""; else L="EMM_LIB_PATH=build/libemm_$v.so"; fi
  echo "== $v"
  env $L timeout 300 python tools/win_probe.py 2>&1 | tail -4
  env $L timeout 300 python tools/attn_bench.py 2>&1 | grep "win"
done
