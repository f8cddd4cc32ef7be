#!/bin/bash
# memcheck over the attention kernels with the work-queue scheduler, and the
# racecheck case that failed a numerics assertion under the tool
export PYTHONUNBUFFERED=1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest \
  tests/test_attention_gpu.py -q -x 2>&1 | tail -3
timeout 600 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest \
  tests/test_attention_gpu.py -q -k "80" 2>&1 | grep -E "FAILED|passed|failed|RACECHECK|Error|assert" | head -20
bash tools/gpu_r02_k1_ncu.sh
