#!/bin/bash
# memcheck over the kernels changed in round 2 (K1 hashes / digests + pixel
# identity path, attention metadata prefetch, K6 transports), then the
# windowed-attention probe
export PYTHONUNBUFFERED=1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest \
  tests/test_hash_gpu.py tests/test_attention_gpu.py -q -x 2>&1 | tail -4
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest \
  tests/test_fullshape_gpu.py -q -x -k "attention" 2>&1 | tail -4
timeout 300 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest \
  tests/test_attention_gpu.py -q -x -k "80" 2>&1 | tail -4
timeout 300 python tools/win_probe.py
