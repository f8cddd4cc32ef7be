#!/bin/bash
# FMNMX3 row max (ATT_MAX3=1, default) vs two-input FMNMX (build/libemm_nomax3.so)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_attention_gpu.py -x -q 2>&1 | tail -2 > gpurun_out/max3_tests.txt
for rep in 1 2; do for v in nomax3 new; do
  if [ $v = new ]; then lib=paper_2507_10069_b200/libemm.so; else lib=build/libemm_$v.so; fi
  echo "== $v (rep $rep)"
  EMM_LIB_PATH=$lib timeout 300 python tools/attn_bench.py 2>&1
done; done > gpurun_out/max3_ab.txt
python tools/win_probe.py > gpurun_out/max3_win.txt 2>&1 || true
