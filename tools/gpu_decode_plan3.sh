#!/bin/bash
# the bench's decode leg with each decode-attention variant
mkdir -p gpurun_out
for v in old o40 o40pre; do
  EMM_LIB_PATH=build/libemm_$v.so timeout 600 python tools/decode_leg_probe.py c3 > gpurun_out/decode_leg_$v.txt 2> gpurun_out/decode_leg_$v.err
done
