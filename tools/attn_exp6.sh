#!/bin/bash
# work-queue scheduling of the pair attention kernel (EMM_ATT_DYN=1, default) vs round-robin
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_fullshape_gpu.py -q -x -k "attention or attn" 2>&1 | tail -2
for d in 0 1 0 1; do
  echo "== EMM_ATT_DYN=$d"
  EMM_ATT_DYN=$d timeout 300 python tools/attn_bench.py 2>&1 | grep -v "vit-clip\|win"
done
EMM_ATT_DYN=1 timeout 600 python tools/fa4_compare.py 2>&1 | grep -v Warn | grep -v warn
