#!/bin/bash
# K1 / K2 launch list with DRAM bytes (ncu, serialised) over tools/dataplane_bench.py
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"block_hash|pixel_|prefix_match" --csv \
  --log-file gpurun_out/launches_k1.csv python tools/dataplane_bench.py > gpurun_out/launches_k1.log 2>&1
python tools/launch_summary.py gpurun_out/launches_k1.csv --out gpurun_out/ncu_k1_k2.json \
  --source "ncu launch list of tools/dataplane_bench.py (K1 block hashes / pixel digests, K2 match)" > /dev/null
cat gpurun_out/ncu_k1_k2.json
