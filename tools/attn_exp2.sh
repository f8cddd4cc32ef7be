#!/bin/bash
# attention variants (tools/build_variant.sh) on the microbench shapes; each
# line: variant, order, then attn_bench output
for v in base pa p7 pap6 pap7; do
  if [ $v = base ]; then L=""; else L="EMM_LIB_PATH=build/libemm_$v.so"; fi
  for o in tile head; do
    if [ $v != base ] && [ $o = head ]; then continue; fi
    echo "== $v order=$o"
    env $L EMM_ATT_ORDER=$o timeout 300 python tools/attn_bench.py 2>&1 | grep -v "^c2\|^long\|win"
  done
done
# one full ncu set of the hd-80 ViT kernel per packing variant
for v in base pa; do
  if [ $v = base ]; then L=""; else L="EMM_LIB_PATH=build/libemm_$v.so"; fi
  env $L timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 \
    -o gpurun_out/attn_vit80_$v python tools/attn_one.py vit80 > gpurun_out/attn_ncu_vit80_$v.log 2>&1
done
