timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 300 python tools/gemm_stream_bench.py 40 64 > gpurun_out/gemm_stream.txt 2>&1; cat gpurun_out/gemm_stream.txt
for w in ours fa4; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd|flash|kernel" -s 3 -c 1 -o gpurun_out/cmp_$w python tools/fa4_one.py $w c3-batch > gpurun_out/cmp_$w.log 2>&1
done
ls gpurun_out/cmp_*
