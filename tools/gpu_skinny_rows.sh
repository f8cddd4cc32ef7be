#!/bin/bash
# split-K reduction in contiguous 16-row passes: correctness, A/B vs the previous build
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_skinny_gpu.py tests/test_gemm_gpu.py tests/test_decode_gpu.py -x -q 2>&1 | tail -3 > gpurun_out/skrows_tests.txt
for v in skold new; do
  if [ $v = new ]; then lib=paper_2507_10069_b200/libemm.so; else lib=build/libemm_$v.so; fi
  echo "== $v"
  EMM_LIB_PATH=$lib timeout 300 python tools/gemm_stream_bench.py 40 64 2>&1 | grep -E "qkv|  o |down|gate"
  for B in 40 64; do EMM_LIB_PATH=$lib timeout 300 python tools/decode_probe.py qwen-7b $B 4400 2>&1 | grep -E "graph replay"; done
  EMM_LIB_PATH=$lib timeout 300 python tools/decode_probe.py qwen-7b 64 profiles/r02/decode_leg_step64_lens.json 2>&1 | grep -E "graph replay"
  EMM_LIB_PATH=$lib timeout 120 python tools/skinny_prof.py 64 3584 3584 2>&1 | tail -8 | grep -E "published|all_arr|epi_done"
done > gpurun_out/skrows_ab.txt 2>&1
EMM_LIB_PATH=build/libemm_skold.so timeout 600 python tools/decode_leg_probe.py c3 > gpurun_out/decode_leg_skold.txt 2>&1
timeout 600 python tools/decode_leg_probe.py c3 > gpurun_out/decode_leg_skrows.txt 2>&1
