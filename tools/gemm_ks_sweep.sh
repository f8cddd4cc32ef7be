#!/bin/bash
# decode GEMMs streamed from HBM (tools/gemm_stream_bench.py) under forced split counts
for ks in 0 2 4 8 12 16; do
  echo "== EMM_GEMM_KS=$ks"
  EMM_GEMM_KS=$ks timeout 300 python tools/gemm_stream_bench.py 64 2>&1 | grep -v gate_up
done
