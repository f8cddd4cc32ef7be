#!/bin/bash
timeout 900 python -m pytest tests/test_attention_gpu.py -q -x 2>&1 | tail -1
timeout 300 python tools/attn_bench.py 2>&1 | grep win
EMM_LIB_PATH=build/libemm_p1.so timeout 300 python tools/attn1_prof.py
timeout 600 ncu --nvtx --nvtx-include win/ --set full --clock-control none --import-source on -c 1 \
  -o gpurun_out/win_tc1 python tools/win_one.py > gpurun_out/win_tc1.log 2>&1
ls -la gpurun_out/win_tc1*
