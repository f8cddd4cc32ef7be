#!/bin/bash
timeout 900 python -m pytest tests/test_gemm_gpu.py -q -x 2>&1 | tail -1
for v in "0 3" "1 2" "1 3" "1 4" "0 3" "1 2" "1 3" "1 4"; do set -- $v
  echo "== EMM_GEMM_TAIL_SPLIT=$1 EMM_GEMM_TAIL_MAXS=$2"
  EMM_GEMM_TAIL_SPLIT=$1 EMM_GEMM_TAIL_MAXS=$2 timeout 300 python tools/gemm_tail_bench.py
done
