#!/bin/bash
# length-aware decode attention plan: parity, old-vs-new kernel, the bench's decode leg
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_decode_gpu.py -q -x 2>&1 | tail -3 > gpurun_out/dp_pytest.txt
echo "== old (splits from the longest row)" > gpurun_out/dp_bench.txt
EMM_LIB_PATH=build/libemm_old.so timeout 300 python tools/decode_bench.py >> gpurun_out/dp_bench.txt 2>&1
echo "== new (per-request splits, persistent)" >> gpurun_out/dp_bench.txt
timeout 300 python tools/decode_bench.py >> gpurun_out/dp_bench.txt 2>&1
timeout 600 python tools/decode_leg_probe.py c3 > gpurun_out/decode_leg_new.txt 2> gpurun_out/decode_leg_new.err
cat gpurun_out/dp_pytest.txt
