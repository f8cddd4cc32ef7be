#!/bin/bash
mkdir -p gpurun_out
( for B in 40 64; do
  echo "== skinny B=$B"; timeout 300 python tools/decode_probe.py qwen-7b $B 4400 2>&1 | tail -12
  echo "== tile kernel B=$B"; EMM_GEMM_SKINNY=0 timeout 300 python tools/decode_probe.py qwen-7b $B 4400 2>&1 | tail -12
done ) 2>&1 | tee gpurun_out/skinny_decode.txt
