for spl in 1 2 4 8; do
  echo "== gather spl=$spl"
  python tools/profile_search.py --m 64 128 256 512 1024 --reps 3 --path 2 --spl $spl 2>&1 | grep -v "rep=0" | awk '{print $1, $5, $6, $7}'
done > gpurun_out/exp.txt 2>&1
