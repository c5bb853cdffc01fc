timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for cfgs in "15360 2" "16384 2" "32768 2"; do
  set -- $cfgs
  echo "== tile=$1 stages=$2"
  python tools/profile_search.py --m 8 16 32 64 --reps 3 --tile $1 --stages $2 2>&1 | grep "rep=2"
done
python tools/profile_search.py --m 128 256 512 1024 --reps 3 2>&1 | grep "rep=2"
