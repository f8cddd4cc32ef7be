#!/bin/bash
# session-4 evidence: default bench line; one recorded 64-request decode step of the
# bench's leg (mixed lengths): launch list + ncu --set full of the decode attention
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench_s4.json 2> gpurun_out/bench_s4.err
N="ncu --nvtx --nvtx-include prof/ --clock-control none"
D="python tools/decode_probe.py qwen-7b 64 profiles/r02/decode_leg_step64_lens.json --ncu"
timeout 600 $N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/launches_decode_s4.csv $D > gpurun_out/launches_decode_s4.log 2>&1
python tools/launch_summary.py gpurun_out/launches_decode_s4.csv --out gpurun_out/launch_shares_decode_s4.json \
  --source "ncu launch list of one recorded decode-leg step (64 requests, mixed lengths; tools/decode_probe.py)" > /dev/null
timeout 600 $N --set full --import-source on -k regex:decode_attn_kernel -c 1 \
  -o gpurun_out/dec_attn_s4 $D > gpurun_out/dec_attn_s4.log 2>&1
ncu -i gpurun_out/dec_attn_s4.ncu-rep --page raw --csv > gpurun_out/dec_attn_s4_raw.csv 2>/dev/null
