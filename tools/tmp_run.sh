P=paper_2310_15711_b200
for lib in prev so; do
  if [ $lib = prev ]; then export HC_LIB=$PWD/$P/libhc_prev.so; else export HC_LIB=$PWD/$P/libhc.so; fi
  echo "== $HC_LIB"
  python tools/batch_bench.py --config C2 --ms 16 32 64 128 256 2>&1 | tail -5 | awk '{print $1, $9, $10, $11}'
  python tools/batch_bench.py --config C4 --ms 16 64 2>&1 | tail -2 | awk '{print $1, $9, $10, $11}'
done
