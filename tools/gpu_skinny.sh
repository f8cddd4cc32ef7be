#!/bin/bash
# decode-size GEMM kernel: correctness, then the weight-stream benchmark
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_skinny_gpu.py tests/test_gemm_gpu.py -x -q 2>&1 | tail -15 > gpurun_out/skinny_tests.txt
cat gpurun_out/skinny_tests.txt
timeout 300 python tools/gemm_stream_bench.py 1 16 40 64 2>&1 | tee gpurun_out/skinny_stream.txt
timeout 120 python tools/skinny_prof.py 40 3584 3584 | tail -11
timeout 120 python tools/skinny_prof.py 40 37888 3584 glu | tail -11
