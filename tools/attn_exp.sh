for x in 0 1 2 3; do
  if [ $x = 0 ]; then L=""; else L="EMM_LIB_PATH=build/libemm_x$x.so"; fi
  echo "== mode $x"; env $L python tools/attn_bench.py 2>&1 | head -2
done
