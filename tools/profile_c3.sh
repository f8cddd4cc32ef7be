#!/bin/bash
# Round evidence at the headline config (C3, Qwen2.5-VL-7B shape), run under gpurun:
#  bench line, launch list of one representative batch (NVTX range "prof"),
#  ncu --set full on the top kernels of that batch.
#  usage: tools/profile_c3.sh [full]   (without "full": bench + launch list only)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
P="python tools/profile_step.py --warm 6 --batch 6"
N="ncu --nvtx --nvtx-include prof/ --clock-control none"
timeout 600 $N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/launches_c3.csv $P > gpurun_out/launches_c3.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c3.csv --out gpurun_out/launch_shares_c3.json \
  --traffic-out gpurun_out/ncu_summary.json \
  --source "ncu launch list of one C3 batch (tools/profile_step.py --warm 6 --batch 6)" > /dev/null
[ "$1" = "full" ] || exit 0
timeout 600 $N --set full --import-source on -k regex:gemm_bf16 -s 171 -c 4 \
  -o gpurun_out/c3_gemm_dec $P > gpurun_out/c3_gemm_dec.log 2>&1
timeout 600 $N --set full --import-source on -k regex:gemm_bf16 -s 33 -c 4 \
  -o gpurun_out/c3_gemm_vit $P > gpurun_out/c3_gemm_vit.log 2>&1
timeout 600 $N --set full --import-source on -k regex:attn_fwd -s 42 -c 1 \
  -o gpurun_out/c3_attn_dec $P > gpurun_out/c3_attn_dec.log 2>&1
timeout 600 $N --set full --import-source on -k regex:attn_fwd -s 7 -c 1 \
  -o gpurun_out/c3_attn_vitfull $P > gpurun_out/c3_attn_vitfull.log 2>&1
timeout 600 $N --set full --import-source on -k regex:attn_fwd -s 0 -c 1 \
  -o gpurun_out/c3_attn_vitwin $P > gpurun_out/c3_attn_vitwin.log 2>&1
timeout 600 $N --set full -k regex:kv_copy -c 2 \
  -o gpurun_out/c3_kvcopy $P > gpurun_out/c3_kvcopy.log 2>&1
ls -la gpurun_out | tail -20
# decode step (Qwen2-7B shape, 64 requests x 4400 context): launch list + full sets
D="python tools/decode_probe.py qwen-7b 64 4400 --ncu"
timeout 600 $N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/launches_decode.csv $D > gpurun_out/launches_decode.log 2>&1
python tools/launch_summary.py gpurun_out/launches_decode.csv --out gpurun_out/launch_shares_decode.json \
  --source "ncu launch list of one decode step (tools/decode_probe.py qwen-7b 64 4400)" > /dev/null
timeout 600 $N --set full --import-source on -k regex:decode_attn_kernel -c 1 \
  -o gpurun_out/dec_attn $D > gpurun_out/dec_attn.log 2>&1
timeout 600 $N --set full --import-source on -k regex:gemm_bf16 -c 4 \
  -o gpurun_out/dec_gemm $D > gpurun_out/dec_gemm.log 2>&1
ls -la gpurun_out | tail -30
