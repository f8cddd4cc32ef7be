#!/bin/bash
# decode GEMMs streamed from HBM with 1 / 2 / 4 K atoms per stage (EMM_GEMM_KA),
# correctness first (split-K GEMM + decode tests under each setting)
for ka in 1 2 4; do
  echo "== EMM_GEMM_KA=$ka"
  EMM_GEMM_KA=$ka timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_decode_gpu.py -q -x 2>&1 | tail -2
  EMM_GEMM_KA=$ka timeout 300 python tools/gemm_stream_bench.py 40 64 2>&1 | grep -v gate_up
done
