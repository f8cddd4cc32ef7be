#!/bin/bash
mkdir -p gpurun_out
( for k in 0 1 2 3 4 8; do echo "== EMM_SKINNY_KS=$k"; EMM_SKINNY_KS=$k timeout 200 python tools/gemm_stream_bench.py 40 2>&1 | grep -v gate_up; done ) 2>&1 | tee gpurun_out/skinny_ks.txt
