#!/bin/bash
# ncu evidence for the round (run under gpurun from the repo root)
set -x
mkdir -p gpurun_out
ARGS="--steps 1 --warmup 1 --no-e2e --no-ttft --no-cpu"
# 1) launch list of one bench step (serialised, cold cache: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3700 -c 3300 --csv \
  --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/launches_bench.log 2>&1
# 2) full sets: 4 GEMMs of one decoder layer (qkv, o, gate/up+SwiGLU, down)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_tc \
  -s 1200 -c 4 -o gpurun_out/gemm_full python bench.py $ARGS > gpurun_out/gemm_full.log 2>&1
# 3) attention (decoder, causal over cached prefix) and the KV gather
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd \
  -s 300 -c 2 -o gpurun_out/attn_full python bench.py $ARGS > gpurun_out/attn_full.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:kv_copy_rows \
  -s 2 -c 1 -o gpurun_out/kvcopy_full python bench.py $ARGS > gpurun_out/kvcopy_full.log 2>&1
ls -la gpurun_out
