timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for cfgs in "24576 3" "16384 4" "28672 3" "20480 4"; do
  set -- $cfgs
  for d in 3 0; do
  echo "== tile=$1 stages=$2 debug=$d"
  python tools/profile_search.py --m 8 16 32 64 128 --reps 3 --tile $1 --stages $2 --path 1 --debug $d 2>&1 | grep "rep=2"
  done
done
