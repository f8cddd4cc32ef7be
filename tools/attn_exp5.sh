#!/bin/bash
# exp2 on the FMA pipe for 1/16 (pm1) or 1/8 (pm2: FA4's middle-fragment pattern, pm3: spread)
for v in base pm1 pm2 pm3 base pm1 pm2 pm3; do
  if [ $v = base ]; then L=""; else L="EMM_LIB_PATH=build/libemm_$v.so"; fi
  echo "== $v"
  env $L timeout 300 python tools/attn_bench.py 2>&1 | grep -v "^c2\|^vit-clip\|win"
done
