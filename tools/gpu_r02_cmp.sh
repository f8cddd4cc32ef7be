for w in ours fa4; do
  for c in c3-batch vit-qwen-full; do
    timeout 600 ncu --nvtx --nvtx-include cmp/ --set full --clock-control none --import-source on \
      -c 4 -o gpurun_out/cmp_${w}_$c python tools/fa4_one.py $w $c > gpurun_out/cmp_${w}_$c.log 2>&1
  done
done
ls gpurun_out/cmp_*
