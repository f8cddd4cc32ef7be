#!/bin/bash
# decode-size GEMM kernel: correctness, then the weight-stream benchmark and the decode step
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_skinny_gpu.py tests/test_gemm_gpu.py tests/test_decode_gpu.py -x -q 2>&1 | tail -5 > gpurun_out/skinny_tests.txt
cat gpurun_out/skinny_tests.txt
timeout 300 python tools/gemm_stream_bench.py 40 64 2>&1 | tee gpurun_out/skinny_stream.txt
for B in 40 64; do timeout 300 python tools/decode_probe.py qwen-7b $B 4400 2>&1 | grep -E "step|graph replay"; done | tee gpurun_out/skinny_decode3.txt
timeout 120 python tools/skinny_prof.py 40 37888 3584 glu | tail -16 | grep -E "acc_ready|epi_done|c0_|c1_"
timeout 120 python tools/skinny_prof.py 40 3584 3584 | tail -16 | grep -E "acc_ready|all_arr|epi_done"
