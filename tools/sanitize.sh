#!/bin/bash
# compute-sanitizer memcheck over the kernel-level GPU tests (run under gpurun)
export PYTHONUNBUFFERED=1
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest \
  tests/test_hash_gpu.py tests/test_decode_gpu.py -q -x -k "not cross_model and not full_recompute"
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest \
  tests/test_attention_gpu.py tests/test_index_gpu.py -q -x
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest \
  tests/test_gemm_gpu.py tests/test_cross_gpu.py tests/test_model_gpu.py -q -x \
  -k "not 8192 and not 4096-11008 and not 32000"
