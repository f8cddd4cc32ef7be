#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/decode_leg_probe.py c3 > gpurun_out/decode_leg_o40.txt 2> gpurun_out/decode_leg_o40.err
python - <<'PY'
import json
log = json.load(open("gpurun_out/decode_leg_c3.json"))
big = [r for r in log if r[0] == 64]
json.dump(big[len(big) // 2][3], open("gpurun_out/leg_step64.json", "w"))
PY
timeout 300 python tools/decode_probe.py qwen-7b 64 gpurun_out/leg_step64.json > gpurun_out/dprobe_leg64.txt 2>&1
timeout 600 ncu --nvtx --nvtx-include prof/ --metrics gpu__time_duration.sum,dram__bytes_read.sum --csv \
  python tools/decode_probe.py qwen-7b 64 gpurun_out/leg_step64.json --ncu > gpurun_out/dprobe_leg64_ncu.csv 2> gpurun_out/dprobe_ncu.err
