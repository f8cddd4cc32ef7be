#!/bin/bash
for v in base pair0 epi2 base; do
  case $v in base) L="";; pair0) L="EMM_GEMM_PAIR=0";; epi2) L="EMM_LIB_PATH=build/libemm_epi2.so";; esac
  echo "== $v"
  env $L timeout 300 python tools/gemm_vit_bench.py 2>&1
done
