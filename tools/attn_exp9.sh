#!/bin/bash
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_fullshape_gpu.py -q -x -k "attention or attn or window or work_queue" 2>&1 | tail -1
timeout 300 python tools/win_probe.py 2>&1 | tail -4
timeout 300 python tools/attn_bench.py 2>&1
EMM_LIB_PATH=build/libemm_p1.so timeout 300 python tools/attn1_prof.py
