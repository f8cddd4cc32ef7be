#!/bin/bash
# attention kernel evidence: microbench + one full-set ncu capture per case
mkdir -p gpurun_out
python tools/attn_bench.py > gpurun_out/attn_bench.txt 2>&1
for c in ${CASES:-qwen vit80}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 \
    -o gpurun_out/attn_$c python tools/attn_one.py $c > gpurun_out/attn_ncu_$c.log 2>&1
done
cat gpurun_out/attn_bench.txt
