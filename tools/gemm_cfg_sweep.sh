#!/bin/bash
# decode GEMM configurations (HBM-streamed weights): BN=64 vs 128 split paths, split counts
for cfg in "EMM_GEMM_SPLITK_BN64=1" "EMM_GEMM_SPLITK_BN64=0" "EMM_GEMM_SPLITK_BN64=0 EMM_GEMM_KS=3" "EMM_GEMM_SPLITK_BN64=0 EMM_GEMM_KS=4" "EMM_GEMM_SPLITK_BN64=0 EMM_GEMM_KA=4" "EMM_GEMM_KA=4"; do
  echo "== $cfg"
  env $cfg timeout 300 python tools/gemm_stream_bench.py 64 2>&1 | grep -v gate_up
done
