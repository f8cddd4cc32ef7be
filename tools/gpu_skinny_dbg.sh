#!/bin/bash
mkdir -p gpurun_out
( echo "== default"; timeout 200 python tools/gemm_stream_bench.py 16 40 64
  echo "== EMM_SKINNY_DBG=1 (no epilogue)"; EMM_SKINNY_DBG=1 timeout 200 python tools/gemm_stream_bench.py 16 40 64 ) 2>&1 | grep -v cublas_x | tee gpurun_out/skinny_dbg.txt
