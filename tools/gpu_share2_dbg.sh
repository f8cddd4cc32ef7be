#!/bin/bash
# 2 ranks sharing cuda:0: with the skinny decode GEMMs (default) and without (EMM_GEMM_SKINNY=0)
mkdir -p gpurun_out
for sk in 0 1; do
( while true; do nvidia-smi --query-gpu=utilization.gpu,clocks.sm,power.draw --format=csv,noheader; sleep 20; done ) > gpurun_out/share2_util_$sk.txt 2>&1 &
MON=$!
EMM_GEMM_SKINNY=$sk EMM_DUMP_AFTER=100 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 2951$sk bench.py --gpus 2 --share-gpu --steps 1 --warmup 1 --no-cpu --no-decode \
  > gpurun_out/share2_dbg_$sk.json 2> gpurun_out/share2_dbg_$sk.err
echo "skinny=$sk rc=$?"
kill $MON
done
