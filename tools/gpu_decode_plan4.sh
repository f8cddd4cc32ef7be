#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/decode_probe.py qwen-7b 64 mixed > gpurun_out/dprobe_mixed.txt 2>&1
EMM_LIB_PATH=build/libemm_old.so timeout 300 python tools/decode_probe.py qwen-7b 64 mixed > gpurun_out/dprobe_mixed_old.txt 2>&1
timeout 300 python tools/decode_probe.py qwen-7b 64 4400 > gpurun_out/dprobe_u64.txt 2>&1
timeout 600 ncu --nvtx --nvtx-include prof/ --metrics gpu__time_duration.sum,dram__bytes_read.sum --csv \
  python tools/decode_probe.py qwen-7b 64 mixed --ncu > gpurun_out/dprobe_mixed_ncu.csv 2> gpurun_out/dprobe_ncu.err
