#!/bin/bash
mkdir -p gpurun_out
( echo "== default"; timeout 200 python tools/gemm_stream_bench.py 40 64
  echo "== EMM_PDL=0"; EMM_PDL=0 timeout 200 python tools/gemm_stream_bench.py 40 64 ) 2>&1 | tee gpurun_out/skinny_pdl.txt
