#!/bin/bash
# round-1 evidence: bench line, launch list of one step, full-set GEMM (decoder layer) + attention + KV copy
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ARGS="--steps 1 --warmup 1 --no-e2e --no-ttft --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3300 -c 3000 --csv \
  --log-file gpurun_out/launches.csv python bench.py $ARGS > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_tc \
  -s 1300 -c 4 -o gpurun_out/gemm_dec python bench.py $ARGS > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd \
  -s 150 -c 1 -o gpurun_out/attn_dec python bench.py $ARGS > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:kv_copy_rows \
  -s 3 -c 2 -o gpurun_out/kvcopy python bench.py $ARGS > /dev/null 2>&1
ls -la gpurun_out
