#!/bin/bash
# N>1 code paths on a one-GPU box: 2 ranks sharing cuda:0 (gloo collectives),
# the elastic-scheduler leg over 2 logical GPUs, and the reference arm under torchrun
mkdir -p gpurun_out
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29517 bench.py --gpus 2 --share-gpu --steps 1 --warmup 1 --no-cpu --no-decode \
  > gpurun_out/bench_share2.json 2> gpurun_out/bench_share2.err
echo "share2 rc=$?"; tail -c 300 gpurun_out/bench_share2.err
timeout 900 python bench.py --engine-gpus 0,0 > gpurun_out/engine_elastic_00.json 2> gpurun_out/engine_elastic_00.err
echo "elastic rc=$?"; tail -c 600 gpurun_out/engine_elastic_00.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29518 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 \
  > gpurun_out/bench_ref2.json 2> gpurun_out/bench_ref2.err
echo "ref2 rc=$?"; tail -c 400 gpurun_out/bench_ref2.json
