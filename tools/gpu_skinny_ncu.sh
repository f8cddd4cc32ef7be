#!/bin/bash
mkdir -p gpurun_out
for M in 64; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_skinny -s 1 -c 1 -o gpurun_out/skinny_plain_$M -f python tools/skinny_one.py $M 37888 3584 > /dev/null 2>&1
ncu -i gpurun_out/skinny_plain_$M.ncu-rep --page details --csv 2>/dev/null | grep -E '"Duration"|"DRAM Throughput"' | head -4
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_skinny -s 1 -c 1 -o gpurun_out/skinny_o_$M -f python tools/skinny_one.py $M 3584 3584 > /dev/null 2>&1
ncu -i gpurun_out/skinny_o_$M.ncu-rep --page details --csv 2>/dev/null | grep -E '"Duration"|"DRAM Throughput"' | head -4
done
