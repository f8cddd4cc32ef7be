#!/bin/bash
# A/B of two library builds (same box, alternating) on the decode step
mkdir -p gpurun_out
( for r in 1 2; do for v in base new; do
  if [ $v = base ]; then export EMM_LIB_PATH=build/libemm_base.so; else unset EMM_LIB_PATH; fi
  for B in 16 40 64 128; do echo "$v r$r B=$B $(timeout 300 python tools/decode_probe.py qwen-7b $B 4400 2>&1 | grep -E 'graph replay|attention_decode' | tr '\n' ' ')"; done
done; done
unset EMM_LIB_PATH
for B in 24 96; do for ns in 0 2 3 4 6 8; do echo "B=$B splits=$ns $(EMM_DECODE_SPLITS=$ns timeout 300 python tools/decode_probe.py qwen-7b $B 2200 2>&1 | grep -E 'attention_decode' | tr '\n' ' ')"; done; done ) 2>&1 | tee gpurun_out/decode_split_ab.txt
