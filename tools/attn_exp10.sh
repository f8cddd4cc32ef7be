#!/bin/bash
# staged, coalesced epilogue stores in the single-tile kernel (ATT1_STAGE_OUT)
EMM_LIB_PATH=build/libemm_so.so timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_fullshape_gpu.py -q -x -k "attention or attn or window or work_queue" 2>&1 | tail -1
for v in base so base so; do
  if [ $v = base ]; then L=""; else L="EMM_LIB_PATH=build/libemm_$v.so"; fi
  echo "== $v"; env $L timeout 300 python tools/win_probe.py 2>&1 | tail -3
done
EMM_LIB_PATH=build/libemm_sop.so timeout 300 python tools/attn1_prof.py
